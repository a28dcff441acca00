# round-2 call J2: interleaved A/B of split_producer / bn384 (3 rounds, same box)
O=gpurun_out/r2j2; mkdir -p $O
for r in 1 2 3; do
for t in "" "split_producer=0" "bn384=0" "split_producer=0,bn384=0"; do
  timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 30 --tune "$t" >> $O/bench.jsonl 2>> $O/bench.err
done; done
