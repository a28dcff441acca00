#!/bin/bash
# merged two-chain narrow tiles (CCT_TUNE_A_TMEM = 4): parity tests, repeatability, same-box A/B,
# launch lists of both forms
O=gpurun_out/mc; mkdir -p $O
timeout 900 python -m pytest tests/test_merged_chains.py tests/test_stress.py::test_gemm_variants_repeatable -q -x \
    > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
B="--steps 2 --warmup 1 --no-e2e --no-cpu --no-configs"
for t in a_tmem=1 a_tmem=4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$t.csv \
      python bench.py $B --tune $t > $O/ncu_$t.log 2>&1
  python tools/launches.py $O/launches_$t.csv > $O/launches_$t.txt
done
AB_TAG=mc/ab NEWTUNES="none a_tmem=4" bash tools/gpu_ab.sh
