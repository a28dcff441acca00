# round-2 call G: fused backward-weight gather -- parity first (bounded), then times / bench / ncu
O=gpurun_out/r2g; mkdir -p $O
timeout 300 python -m pytest tests/test_gather.py -q -x --timeout 120 -k wgrad > $O/wgrad_tests.log 2>&1; echo "tests rc $?" >> $O/wgrad_tests.log
grep -q "tests rc 0" $O/wgrad_tests.log || exit 0
for g in 1 0; do
  timeout 120 python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 --tune gather=$g >> $O/time.log 2>&1
done
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 >> $O/bench.jsonl 2>> $O/bench.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_bench.log 2>&1; echo "ncu rc $?" >> $O/ncu_bench.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wgrad_gather -c 1 -o $O/gather_wgrad -f python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu rc $?" >> $O/ncu_full.log
timeout 600 python -m pytest tests/test_gather.py tests/test_gpu_parity.py -q --timeout 300 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
