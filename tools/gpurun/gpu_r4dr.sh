#!/bin/bash
# narrow tiles with the deeper A ring (CCT_TUNE_A_TMEM = 5): parity tests, repeatability, same-box A/B,
# launch lists of both forms
O=gpurun_out/dr; mkdir -p $O
timeout 900 python -m pytest tests/test_narrow_ring.py tests/test_stress.py::test_gemm_variants_repeatable -q -x \
    > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
B="--steps 2 --warmup 1 --no-e2e --no-cpu --no-configs"
for t in a_tmem=1 a_tmem=5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$t.csv \
      python bench.py $B --tune $t > $O/ncu_$t.log 2>&1
  python tools/launches.py $O/launches_$t.csv > $O/launches_$t.txt
done
AB_TAG=dr/ab NEWTUNES="none a_tmem=5" bash tools/gpu_ab.sh
