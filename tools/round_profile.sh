#!/bin/bash
# GPU evidence for profiles/: the ncu launch list of the bench step and ncu --set
# full captures of the top kernels, summarised ON the box (the .ncu-rep files are
# large; only text comes back).  Usage: bash tools/round_profile.sh [tests]
set -u
O=gpurun_out/prof
mkdir -p $O
if [ "${1:-}" = "tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -4 $O/smoke.log
  timeout 400 python bench.py > $O/bench.json 2> $O/bench.err; cat $O/bench.json
  timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
fi
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launches.py $O/launches.csv > $O/launches.txt
python tools/gemm_traffic.py $O/launches.csv $O/gemm_traffic.json 15 > /dev/null
R=/tmp/ncu_reps; mkdir -p $R
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm3x|col2im|transpose" -c 6 \
    -o $R/conv2_full python tools/layer_step.py 27 5 96 256 1 2 1 > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm3x|col2im|lower_t1|expand" -c 8 \
    -o $R/conv1_full python tools/layer_step.py 227 11 3 96 4 0 1 > $O/ncu_c1.log 2>&1
python tools/ncu_summary.py $R/conv2_full.ncu-rep "conv2 b=256 training step (auto): fwd GEMM, dy transpose, swapped implicit dgrad, wgrad" > $O/ncu_full_conv2.txt
python tools/ncu_summary.py $R/conv1_full.ncu-rep "conv1 b=256 training step (auto): lower, fwd GEMM, expand, dgrad GEMM, col2im, wgrad" > $O/ncu_full_conv1.txt
cuobjdump -sass paper_1504_04343_b200/_lib/libcct.so | grep -oE "UTCHMMA(\.2CTA)?|UTMALDG\.[A-Z0-9.]+|UTMASTG|UBLKCP[A-Z.0-9]*|LDTM\.x[0-9]+|STTM\.x[0-9]+" | sort | uniq -c | sort -rn > $O/sass_evidence.txt
ls -la $O
