# round-2 call H2: non-swapped implicit backward-data by default -- tests, bench x2, launch list
O=gpurun_out/r2h2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 >> $O/bench.jsonl 2>> $O/bench.err; done
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 --tune dgrad_swap=1 >> $O/bench.jsonl 2>> $O/bench.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_bench.log 2>&1; echo "ncu rc $?" >> $O/ncu_bench.log
