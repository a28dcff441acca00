O=gpurun_out/r3r; mkdir -p $O
timeout 900 python -m pytest tests/test_gather.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc $?" >> $O/tests.log
./tools/hfold_probe 256 > $O/hprobe.log 2>&1
./tools/gather_probe 256 > $O/gprobe.log 2>&1
AB_TAG=r3r/ab VARIANTS="nossa nopace" bash tools/gpu_ab.sh
