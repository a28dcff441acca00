# compute-sanitizer memcheck / synccheck / racecheck over every GEMM instance, the fused conv1
# kernels (incl. the overlapped backward), and the Types 2/3 streaming kernels
O=gpurun_out/r3ze; mkdir -p $O
for t in memcheck synccheck racecheck; do
  timeout 1700 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_cases.py > $O/sanitize_$t.log 2>&1; echo "$t rc $?" >> $O/sanitize_$t.log
done
