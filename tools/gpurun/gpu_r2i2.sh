# round-2 call I2: narrow tiles without the split (two sub-accumulator chains); re-A/B the GEMM variant
# switches on the round-2 build (step time, same box)
O=gpurun_out/r2i2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_stress.py tests/test_layout.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
grep -q "tests rc 0" $O/tests.log || exit 0
timeout 120 python tools/pass_time.py --layer conv2 --pass dgrad --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv2 --pass dgrad --layout 1 --reps 20 --tune dgrad_swap=1 >> $O/time.log 2>&1
for t in "" "dgrad_swap=1" "split_producer=0" "a_tmem_wide=0" "bn384=0" "streamk=0" "chain2=0" "cta_pairs=1" "" "dgrad_swap=1"; do
  timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 --tune "$t" >> $O/bench.jsonl 2>> $O/bench.err
done
