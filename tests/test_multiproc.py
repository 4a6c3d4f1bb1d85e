"""World-size-2 `gloo` test of the multi-GPU host logic (CPU): every rank
derives the same layer ownership and kernel offsets from its own plan, writes
only the layers it owns into its rank-major segment, and one all-gather gives
every rank every layer at the offsets a single-rank plan would read them."""
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


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2601_13776_b200 as orth
        from paper_2601_13776_b200.dist import batch_shard, gather_kernels
        cfg = configs.cfg3()
        plan = orth.Plan(cfg, device=-1, rank=rank, world=world)
        seg = orth.orth_plan_query(plan.h, "KERNEL_SEGMENT_F32")
        kbuf = torch.zeros(plan.kf32_numel)
        owned = 0
        for l, info in enumerate(plan.layer_info):
            if info["owner"] == rank:       # stand-in for orth_compose_kernel's writes
                kbuf[info["kf32_off"]: info["kf32_off"] + info["numel"]] = l + 1 + torch.arange(info["numel"]) * 1e-6
                owned += 1
        gather_kernels(plan, kbuf, seg)
        ok = True
        for l, info in enumerate(plan.layer_info):
            want = l + 1 + torch.arange(info["numel"]) * 1e-6
            ok &= bool(torch.equal(kbuf[info["kf32_off"]: info["kf32_off"] + info["numel"]], want))
        b, e = batch_shard(256, rank, world)
        q.put((rank, ok, owned, (b, e)))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover
        q.put((rank, repr(ex), 0, None))


def test_sharded_construction_allgather_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, ok, owned, shard in res:
        assert ok is True, (rank, ok)
        assert owned > 0
    assert res[0][3] == (0, 128) and res[1][3] == (128, 256)
    assert res[0][2] + res[1][2] == len(configs.cfg3())
