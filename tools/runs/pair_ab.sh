set -x
ORTH_EXPERIMENTAL=1 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pair_build.log 2>&1
for v in 0 1; do
  if [ $v = 1 ]; then export ORTH_CONV_PAIR=1; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pair_ab_$v.json 2> gpurun_out/pair_ab_$v.err
  echo "v=$v rc=$?"
done
