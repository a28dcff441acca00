# round-2 evidence E1: full bench (value, e2e, CPU baseline, configs), reference arm, launch list,
# ncu --set full of the step's top kernels
O=gpurun_out/r2e1; mkdir -p $O
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err; echo "bench rc $?" >> $O/bench_full.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc $?" >> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_bench.log 2>&1; echo "ncu rc $?" >> $O/ncu_bench.log
# one --set full capture per top kernel of the step (warm-up step skipped: --launch-skip)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm3xtf32 --launch-skip 15 --launch-count 15 -o $O/step_gemms -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_full_gemm.log 2>&1; echo "ncu rc $?" >> $O/ncu_full_gemm.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gather_kernel|hfold_kernel|vfold" --launch-skip 4 --launch-count 4 -o $O/step_conv1 -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_full_conv1.log 2>&1; echo "ncu rc $?" >> $O/ncu_full_conv1.log
