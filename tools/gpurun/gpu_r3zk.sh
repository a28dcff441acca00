O=gpurun_out/${TAG:-r3zk}; mkdir -p $O
for r in 1 2 3; do
  (cd abtest/old && python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20) >> $O/pt_old.log 2>&1
  python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 >> $O/pt_new.log 2>&1
done
timeout 900 python -m pytest tests/test_gather.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc $?" >> $O/tests.log
timeout 1700 compute-sanitizer --tool racecheck --print-limit 200 --kernel-name-exclude kns=gemm3xtf32 python tools/sanitize_cases.py > $O/racecheck_nongemm.log 2>&1; echo "rc $?" >> $O/racecheck_nongemm.log
