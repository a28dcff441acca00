# round-2 call Y: lift loop order per type
O=gpurun_out/r2y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py tests/test_ext.py tests/test_layout.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
grep -q "tests rc 0" $O/tests.log || exit 0
timeout 1500 python tools/sweep.py --out $O/sweep.jsonl --extra "27,5,96,256,1,2;13,3,256,384,1,1;13,3,384,384,1,1;13,3,384,256,1,1" > $O/sweep.log 2>&1; echo "sweep rc $?" >> $O/sweep.log
