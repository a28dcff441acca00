# round-2 call N: gather before the A-slot wait (fwd merged + wgrad)
O=gpurun_out/r2n; mkdir -p $O
timeout 300 python -m pytest tests/test_gather.py -q -x --timeout 120 > $O/gather_tests.log 2>&1; echo "tests rc $?" >> $O/gather_tests.log
grep -q "tests rc 0" $O/gather_tests.log || exit 0
for i in 1 2; do
timeout 120 python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 20 >> $O/time.log 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:fwd_gather -c 1 -o $O/gather_fwd -f python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 1 > $O/ncu_full2.log 2>&1; echo "ncu rc $?" >> $O/ncu_full2.log
