O=gpurun_out/r3p; mkdir -p $O
timeout 900 python -m pytest tests/test_gather.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc $?" >> $O/tests.log
./tools/gather_probe 256 > $O/probe.log 2>&1
AB_TAG=r3p/ab bash tools/gpu_ab.sh
