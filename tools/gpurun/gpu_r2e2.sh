# round-2 evidence E2: compute-sanitizer (memcheck, synccheck, racecheck) incl. the fused conv1 kernels; hang soak
O=gpurun_out/r2e2; mkdir -p $O
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_cases.py > $O/sanitize_$t.log 2>&1; echo "$t rc $?" >> $O/sanitize_$t.log
done
for i in $(seq 1 30); do timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e --no-configs > $O/soak_$i.json 2>/dev/null; echo "soak $i rc $?" >> $O/soak.log; done
