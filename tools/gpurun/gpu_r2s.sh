# round-2 call S: hfold v3 (A via TMEM, 6-deep raw ring)
O=gpurun_out/r2u; mkdir -p $O
timeout 300 python -m pytest tests/test_gather.py -q -x --timeout 120 -k hfold > $O/hfold_tests.log 2>&1; echo "tests rc $?" >> $O/hfold_tests.log
grep -q "tests rc 0" $O/hfold_tests.log || exit 0
for i in 1 2; do
timeout 120 python tools/pass_time.py --layer conv1 --pass dgrad --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass dgrad --layout 1 --reps 20 --tune gather=0 >> $O/time.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/dgrad_launches.csv python tools/pass_time.py --layer conv1 --pass dgrad --layout 1 --reps 1 > $O/ncu_l.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:conv_dgrad_hfold -c 1 -o $O/hfold -f python tools/pass_time.py --layer conv1 --pass dgrad --layout 1 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu rc $?" >> $O/ncu_full.log
