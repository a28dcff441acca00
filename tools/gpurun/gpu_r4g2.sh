#!/bin/bash
# conv1 forward: merged (default) vs 6-MMA form (CCT_TUNE_GATHER = 2) with the 600 ns epilogue pause
O=gpurun_out/g2; mkdir -p $O
B="--steps 2 --warmup 1 --no-e2e --no-cpu --no-configs"
for r in 1 2; do
for t in gather=1 gather=2; do
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:conv_fwd_gather --csv \
      --log-file $O/${t}_$r.csv python bench.py $B --tune $t > $O/ncu_${t}_$r.log 2>&1
done
done
