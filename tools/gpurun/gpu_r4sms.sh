#!/bin/bash
# conv1 forward gather with A_small in shared memory (CCT_TUNE_GATHER = 4): parity, repeatability,
# ncu kernel times of both forms in the bench step, same-box A/B of the step
O=gpurun_out/sms; mkdir -p $O
timeout 900 python -m pytest tests/test_gather.py tests/test_stress.py::test_gemm_variants_repeatable -q -x \
    > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
B="--steps 2 --warmup 1 --no-e2e --no-cpu --no-configs"
for r in 1 2; do
for t in gather=1 gather=4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_fwd_gather --csv \
      --log-file $O/${t}_$r.csv python bench.py $B --tune $t > $O/ncu_${t}_$r.log 2>&1
done
done
AB_TAG=sms/ab NEWTUNES="none gather=4" bash tools/gpu_ab.sh
