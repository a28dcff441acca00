#!/bin/bash
# conv1 forward gather: kernel-bank ring depth sensitivity (compile-time CCT_FWD_MAX_STAGES caps,
# abtest/stN from tools/build_variant.sh; the product fits 7 stages next to the row stage)
O=gpurun_out/st; mkdir -p $O
B="--steps 2 --warmup 1 --no-e2e --no-cpu --no-configs"
for r in 1 2; do
for v in prod st6 st5 st4 st3; do
  if [ $v = prod ]; then env=""; else env="CCT_LIB_DIR=abtest/$v"; fi
  env $env timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_fwd_gather --csv \
      --log-file $O/${v}_$r.csv python bench.py $B > $O/${v}_$r.log 2>&1
done
done
