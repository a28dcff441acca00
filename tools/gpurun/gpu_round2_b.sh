# round-2 GPU call B: new bench (configs, e2e with D2H, CPU baseline at b=32 + configs[0]),
# reference arm, multi-rank ConvStack test, compute-sanitizer logs, 50-run hang soak.
O=gpurun_out/r2b; mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q --timeout 800 > $O/multigpu.log 2>&1; echo "multigpu rc $?" >> $O/multigpu.log
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc $?"
for t in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_cases.py > $O/sanitize_$t.log 2>&1; echo "$t rc $?" >> $O/sanitize_$t.log
done
for i in $(seq 1 50); do timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e --no-configs > $O/soak_$i.json 2>/dev/null; echo "soak $i rc $?" >> $O/soak.log; done
