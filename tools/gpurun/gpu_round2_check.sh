set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2a/tests.log 2>&1; echo "tests rc $?" >> gpurun_out/r2a/tests.log
for i in 1 2 3 4 5 6; do timeout 240 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2a/bench_$i.json 2> gpurun_out/r2a/bench_$i.err; echo "bench $i rc $?"; done
timeout 600 python bench.py > gpurun_out/r2a/bench_full.json 2> gpurun_out/r2a/bench_full.err; echo "full rc $?"
