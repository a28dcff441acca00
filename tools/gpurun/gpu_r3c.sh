O=gpurun_out/r3c; mkdir -p $O
./tools/hfold_probe 256 > $O/probe.log 2>&1
timeout 900 python -m pytest tests/test_gather.py -q -x --timeout 600 > $O/gather.log 2>&1; echo "rc $?" >> $O/gather.log
