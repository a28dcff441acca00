# round-2 call H: wgrad gather with per-k-block row bases
O=gpurun_out/r2h; mkdir -p $O
timeout 300 python -m pytest tests/test_gather.py -q -x --timeout 120 > $O/gather_tests.log 2>&1; echo "tests rc $?" >> $O/gather_tests.log
grep -q "tests rc 0" $O/gather_tests.log || exit 0
timeout 120 python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 >> $O/time.log 2>&1
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 >> $O/bench.jsonl 2>> $O/bench.err; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wgrad_gather -c 1 -o $O/gather_wgrad -f python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu rc $?" >> $O/ncu_full.log
