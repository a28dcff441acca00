# round-2 call I: wgrad MMA loop (templated M-tiles, one elect per k-block); conv1 dgrad alternatives
O=gpurun_out/r2i; mkdir -p $O
timeout 300 python -m pytest tests/test_gather.py -q -x --timeout 120 > $O/gather_tests.log 2>&1; echo "tests rc $?" >> $O/gather_tests.log
grep -q "tests rc 0" $O/gather_tests.log || exit 0
timeout 120 python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass dgrad --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass dgrad --layout 1 --reps 20 --tune s2d=2 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass dgrad --layout 1 --reps 20 --tune s2d=2,dgrad_swap=0 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 20 --tune gather=0,s2d=2 >> $O/time.log 2>&1
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 >> $O/bench.jsonl 2>> $O/bench.err; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wgrad_gather -c 1 -o $O/gather_wgrad -f python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu rc $?" >> $O/ncu_full.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/dgrad_s2d.csv python tools/pass_time.py --layer conv1 --pass dgrad --layout 1 --reps 1 --tune s2d=2 > $O/ncu_s2d.log 2>&1
