# round-2 GPU call C: full GPU suite (layout, sweep parity, multi-rank), T2/T3 phase sweep, bench
O=gpurun_out/r2c; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
timeout 900 python tools/sweep.py --out $O/sweep.jsonl > $O/sweep.log 2>&1; echo "sweep rc $?" >> $O/sweep.log
timeout 600 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; echo "bench rc $?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_bench.log 2>&1; echo "ncu rc $?" >> $O/ncu_bench.log
