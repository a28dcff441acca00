# round-2 call F: branch-free gather; NHWC stack A/B; full GPU tests
O=gpurun_out/r2f; mkdir -p $O
timeout 300 python tools/pass_time.py --layer conv1 --pass fwd --reps 20 > $O/time.log 2>&1
for lay in nchw nhwc nchw nhwc; do
  timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 --layout $lay >> $O/bench.jsonl 2>> $O/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_nhwc.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-configs --layout nhwc > $O/ncu_bench.log 2>&1; echo "ncu rc $?" >> $O/ncu_bench.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gather -c 1 -o $O/gather_fwd -f python tools/pass_time.py --layer conv1 --pass fwd --reps 1 > $O/ncu_full.log 2>&1; echo "ncu rc $?" >> $O/ncu_full.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
