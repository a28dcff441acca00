#!/bin/bash
# final build: every GPU test, smoke, bench + reference arm, launch list / ncu summaries
# (tools/round_profile.sh), then racecheck / memcheck of the non-GEMM kernels (incl. the
# bulk-store expand) over tools/sanitize_cases.py
PROF_TAG=r2i bash tools/round_profile.sh tests
O=gpurun_out/r2i
timeout 1500 compute-sanitizer --tool racecheck --print-limit 200 --kernel-name-exclude kns=gemm3xtf32 python tools/sanitize_cases.py > $O/racecheck_nongemm.log 2>&1; echo "rc $?" >> $O/racecheck_nongemm.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_cases.py > $O/memcheck.log 2>&1; echo "rc $?" >> $O/memcheck.log
