# round-3 D: hfold linear tiles + fold/backward-weight overlap: parity, then interleaved A/B of the step
O=gpurun_out/r3d; mkdir -p $O
timeout 900 python -m pytest tests/test_gather.py tests/test_stress.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc $?" >> $O/tests.log
for r in 1 2 3; do
  for t in overlap=1 overlap=0; do
    timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu --no-configs --tune $t > $O/bench_${t}_$r.json 2>$O/bench_${t}_$r.err
  done
done
./tools/hfold_probe 256 > $O/probe.log 2>&1
