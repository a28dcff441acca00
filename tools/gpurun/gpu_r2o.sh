# round-2 call O: fwd gather merged (gather=1) vs 6-MMA (gather=2), same box
O=gpurun_out/r2o; mkdir -p $O
timeout 300 python -m pytest tests/test_gather.py -q -x --timeout 120 > $O/gather_tests.log 2>&1; echo "tests rc $?" >> $O/gather_tests.log
for i in 1 2; do for g in 1 2; do
timeout 120 python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 20 --tune gather=$g >> $O/time.log 2>&1
done; done
