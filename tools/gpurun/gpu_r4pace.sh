#!/bin/bash
# conv1 forward gather epilogue pacing sweep: ncu kernel times of conv_fwd_gather_kernel for
# compile-time CCT_FWD_PACE_NS variants (abtest/paceN, tools/build_variant.sh) and the product (300)
O=gpurun_out/pace; mkdir -p $O
B="--steps 2 --warmup 1 --no-e2e --no-cpu --no-configs"
for r in 1 2; do
for v in prod pace0 pace150 pace600 pace1200 pace2400; do
  if [ $v = prod ]; then env=""; else env="CCT_LIB_DIR=abtest/$v"; fi
  env $env timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_fwd_gather --csv \
      --log-file $O/${v}_$r.csv python bench.py $B > $O/${v}_$r.log 2>&1
done
done
