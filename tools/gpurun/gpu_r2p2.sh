# round-2 call P2: e2e with write-combined H2D sources (A/B)
O=gpurun_out/r2p2; mkdir -p $O
for i in 1 2; do for wc in 0 1; do
  timeout 300 python bench.py --no-cpu --no-configs --steps 10 --h2d-wc $wc >> $O/bench.jsonl 2>> $O/bench.err
done; done
