# fused small-channel gather: parity tests, conv1 forward time, ncu of the kernel
O=gpurun_out/gather; mkdir -p $O
timeout 600 python -m pytest tests/test_gather.py -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
timeout 300 python tools/pass_time.py --layer conv1 --pass fwd --reps 20 > $O/time.log 2>&1
timeout 300 python tools/pass_time.py --layer conv1 --pass fwd --reps 20 --tune gather=0 >> $O/time.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gather -c 1 -o $O/gather_fwd -f python tools/pass_time.py --layer conv1 --pass fwd --reps 1 > $O/ncu.log 2>&1; echo "ncu rc $?" >> $O/ncu.log
