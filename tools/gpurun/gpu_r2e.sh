# round-2 call E: warp-uniform MMA / TMA issue (no ELECT waterfall) -- tests, pass times, bench, launch list
O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
for g in 1 0; do
  timeout 300 python tools/pass_time.py --layer conv1 --pass fwd --reps 20 --tune gather=$g >> $O/time.log 2>&1
done
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 >> $O/bench.jsonl 2>> $O/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_bench.log 2>&1; echo "ncu rc $?" >> $O/ncu_bench.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gather -c 1 -o $O/gather_fwd -f python tools/pass_time.py --layer conv1 --pass fwd --reps 1 > $O/ncu_full.log 2>&1; echo "ncu rc $?" >> $O/ncu_full.log
