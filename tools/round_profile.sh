#!/bin/bash
# One gpurun call producing the round's evidence, all under gpurun_out/${PROF_TAG:-prof}/:
# GPU tests, smoke, the full bench line and the reference arm, the ncu launch list of a bench
# step (+ per-kernel summary and the GEMMs' DRAM bytes per launch), ncu --set full captures of
# the step's main GEMMs and fused conv1 kernels (summarised ON the box: the .ncu-rep files are
# large), and the SASS mnemonics that show tcgen05 / TMA.
#   gpurun --timeout 3000 -- 'bash tools/round_profile.sh [tests]'
set -u
O=gpurun_out/${PROF_TAG:-prof}
mkdir -p $O
if [ "${1:-}" = "tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "tests rc $?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
fi
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err; echo "bench rc $?" >> $O/bench_full.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc $?" >> $O/bench_reference.err
# launch list of one step (step 2 of 2: the second half of the list); per-launch times are
# cold-cache and serialised -- the kernels' shares of the step are what carries over
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-configs > $O/ncu_launches.log 2>&1
python tools/launches.py $O/launches.csv > $O/launches.txt
python tools/gemm_traffic.py $O/launches.csv $O/gemm_traffic.json 15 > /dev/null
R=/tmp/ncu_reps; mkdir -p $R
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm3xtf32 --launch-skip 12 --launch-count 12 \
    -o $R/step_gemms -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_full_gemms.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gather_kernel|hfold_kernel|vfold" \
    --launch-skip 4 --launch-count 4 -o $R/step_conv1 -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e \
    --no-configs > $O/ncu_full_conv1.log 2>&1
python tools/ncu_summary.py $R/step_gemms.ncu-rep "the 12 main GEMM launches of one bench step (ncu --set full)" > $O/ncu_full_step_gemms.txt
python tools/ncu_summary.py $R/step_conv1.ncu-rep "conv1 fused kernels of one bench step (ncu --set full)" > $O/ncu_full_step_conv1.txt
cuobjdump -sass paper_1504_04343_b200/_lib/libcct.so | grep -oE "UTCHMMA(\.2CTA)?|UTCQMMA[A-Z0-9.]*|UTMALDG\.[A-Z0-9.]+|UTMASTG|UBLKCP[A-Z.0-9]*|LDTM\.x[0-9]+|STTM\.x[0-9]+" | sort | uniq -c | sort -rn > $O/sass_evidence.txt
ls -la $O
