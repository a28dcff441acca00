# round-2 call M2: chunked fused conv1 test; ncu --set full of the final-default step GEMMs and conv1 kernels
O=gpurun_out/r2m2; mkdir -p $O
timeout 600 python -m pytest tests/test_gather.py -q --timeout 300 -k "workspace_limit" > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm3xtf32 --launch-skip 12 --launch-count 12 -o $O/step_gemms -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_full_gemm.log 2>&1; echo "ncu rc $?" >> $O/ncu_full_gemm.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gather_kernel|hfold_kernel|vfold" --launch-skip 4 --launch-count 4 -o $O/step_conv1 -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-configs > $O/ncu_full_conv1.log 2>&1; echo "ncu rc $?" >> $O/ncu_full_conv1.log
