"""World-size-2/3 `gloo` tests of the multi-GPU host logic (CPU, host-only
plans): every rank derives the same (layer, group) unit ownership and the same
gather / final offsets from its own plan; writing only its own units into its
rank-major gather segment and one all-gather give every rank every unit, and
the unit table's gather -> final copy (what orth_kernels_assemble does on the
device) reproduces, for every layer, the contiguous kernel a single-rank plan
reads.  The device side of the same path (real orth_compose_kernel writes,
orth_kernels_assemble) is tests/test_gpu_sharded.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import configs


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _unit_values(u, numel):
    # a distinct, exactly representable value per (layer, group, element)
    return (u["layer"] * 64 + u["group"] + 1) + torch.arange(numel, dtype=torch.float64) / 2 ** 20


def _worker(rank, world, port, cfg_name, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2601_13776_b200 as orth
        from paper_2601_13776_b200.dist import batch_shard, gather_kernels
        cfg = getattr(configs, cfg_name)()
        plan = orth.Plan(cfg, device=-1, rank=rank, world=world)
        ref = orth.Plan(cfg, device=-1)
        gbuf = torch.zeros(plan.gf32_numel, dtype=torch.float64)
        owned = 0
        for u in plan.units:
            if u["owner"] == rank:       # stand-in for orth_compose_kernel's writes (host-only plan)
                assert rank * plan.seg_f32 <= u["gat_f32"] and u["gat_f32"] + u["numel"] <= (rank + 1) * plan.seg_f32
                gbuf[u["gat_f32"]: u["gat_f32"] + u["numel"]] = _unit_values(u, u["numel"])
                owned += 1
        gather_kernels(gbuf, plan.seg_f32)
        final = torch.zeros(plan.kf32_numel, dtype=torch.float64)
        for u in plan.units:          # orth_kernels_assemble's copy, from the queried unit table
            final[u["fin_f32"]: u["fin_f32"] + u["numel"]] = gbuf[u["gat_f32"]: u["gat_f32"] + u["numel"]]
        ok = plan.kf32_numel == ref.kf32_numel
        for l, info in enumerate(ref.layer_info):   # the single-rank plan's layer offsets
            per = info["numel"] // cfg[l].get("g", 1)
            want = torch.cat([_unit_values(dict(layer=l, group=g), per) for g in range(cfg[l].get("g", 1))])
            ok &= bool(torch.equal(final[info["kf32_off"]: info["kf32_off"] + info["numel"]], want))
        b, e = batch_shard(256, rank, world)
        q.put((rank, ok, owned, (b, e)))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover
        q.put((rank, repr(ex), 0, None))


@pytest.mark.parametrize("cfg_name,world", [("cfg3", 2), ("cfg4", 3)])
def test_sharded_construction_allgather_gloo(cfg_name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, ok, owned, shard in res:
        assert ok is True, (rank, ok)
        assert owned > 0
    n_units = sum(d.get("g", 1) for d in getattr(configs, cfg_name)())
    assert sum(r[2] for r in res) == n_units
    per = (256 + world - 1) // world
    assert [r[3] for r in res] == [(r * per, min(256, (r + 1) * per)) for r in range(world)]
