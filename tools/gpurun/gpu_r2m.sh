# round-2 call M: fwd merged N=2NP MMA + decoupled rings; wgrad gather group per M-tile
O=gpurun_out/r2m; mkdir -p $O
timeout 300 python -m pytest tests/test_gather.py -q -x --timeout 120 > $O/gather_tests.log 2>&1; echo "tests rc $?" >> $O/gather_tests.log
grep -q "tests rc 0" $O/gather_tests.log || exit 0
for i in 1 2; do
timeout 120 python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 20 >> $O/time.log 2>&1
done
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 >> $O/bench.jsonl 2>> $O/bench.err; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wgrad_gather -c 1 -o $O/gather_wgrad -f python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu rc $?" >> $O/ncu_full.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:fwd_gather -c 1 -o $O/gather_fwd -f python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 1 > $O/ncu_full2.log 2>&1; echo "ncu rc $?" >> $O/ncu_full2.log
