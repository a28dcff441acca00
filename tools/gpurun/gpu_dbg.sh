O=gpurun_out/dbg; mkdir -p $O
CCT_LIB_DIR=build/trace timeout 120 python tools/pass_time.py --layer conv1 --pass fwd --reps 1 > $O/trace.out 2> $O/trace.log
timeout 600 python -m pytest tests/test_gather.py -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
timeout 300 python tools/pass_time.py --layer conv1 --pass fwd --reps 20 > $O/time.log 2>&1
