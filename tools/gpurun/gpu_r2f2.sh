# round-2 call F2: vectorized split-K reduce (parity + repeatability tests), e2e copy streams A/B
O=gpurun_out/r2f2; mkdir -p $O
timeout 900 python -m pytest tests/test_stress.py tests/test_gpu_parity.py tests/test_gather.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
grep -q "tests rc 0" $O/tests.log || exit 0
for cs in 1 2 3 1 2 3; do timeout 300 python bench.py --no-cpu --no-configs --steps 10 --copy-streams $cs >> $O/bench.jsonl 2>> $O/bench.err; done
