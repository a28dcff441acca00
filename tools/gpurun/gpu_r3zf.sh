# racecheck restricted to the non-GEMM kernels (the GEMM's two known async-proxy patterns fill the print limit)
O=gpurun_out/${TAG:-r3zf}; mkdir -p $O
timeout 1700 compute-sanitizer --tool racecheck --print-limit 200 --kernel-name-exclude kns=gemm3xtf32 python tools/sanitize_cases.py > $O/racecheck_nongemm.log 2>&1; echo "rc $?" >> $O/racecheck_nongemm.log
timeout 900 python -m pytest tests/test_gather.py -q -x --timeout 600 > $O/gather_tests.log 2>&1; echo "rc $?" >> $O/gather_tests.log
