O=gpurun_out/r3zb; mkdir -p $O
timeout 900 python tools/sweep.py --out $O/sweep.jsonl > $O/sweep.log 2>&1
