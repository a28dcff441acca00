# round-2 call N2: wgrad gather with row-aligned tiles and three row buffers
O=gpurun_out/r2n2; mkdir -p $O
timeout 600 python -m pytest tests/test_gather.py -q -x --timeout 300 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
grep -q "tests rc 0" $O/tests.log || exit 0
for i in 1 2; do timeout 120 python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 >> $O/time.log 2>&1; done
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 >> $O/bench.jsonl 2>> $O/bench.err; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wgrad_gather -c 1 -o $O/wgrad -f python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 1 > $O/ncu.log 2>&1
