#!/bin/bash
# hang / stability soak of the last build: 20 consecutive bench runs of 30 steps each
O=gpurun_out/soak; mkdir -p $O
for i in $(seq 1 20); do
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu --no-configs >> $O/soak.jsonl 2>> $O/soak.err
  echo "run $i rc $?" >> $O/soak_rc.log
done
