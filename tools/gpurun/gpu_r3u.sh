# T2/T3 streaming kernels: parity, ncu of lift / expand, the configs[1] sweep
O=gpurun_out/${TAG:-r3u}; mkdir -p $O; R=/tmp/reps; mkdir -p $R
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "t23 or edge or caffenet or sweep or golden" > $O/tests.log 2>&1; echo "rc $?" >> $O/tests.log
timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x --timeout 800 > $O/tests_sweep.log 2>&1; echo "rc $?" >> $O/tests_sweep.log
for t in 3 2; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"lift|expand" -o $R/le$t -f \
      python tools/layer_step.py 13 3 256 256 1 1 $t > $O/ncu_$t.log 2>&1
  python tools/ncu_summary.py $R/le$t.ncu-rep "T$t lift / expand (n 13, k 3, d = o = 256, b 256)" > $O/le$t.txt
done
[ -z "${NOSWEEP:-}" ] && timeout 900 python tools/sweep.py --out $O/sweep.jsonl > $O/sweep.log 2>&1
