# round-2 call P: configs[1] lowering-type sweep + GEMM rate table on the current build (cost-model re-validation)
O=gpurun_out/r2p; mkdir -p $O
timeout 1500 python tools/sweep.py --out $O/sweep.jsonl > $O/sweep.log 2>&1; echo "sweep rc $?" >> $O/sweep.log
timeout 900 python tools/gemm_bench.py --rate-table > $O/rate_table.json 2> $O/rate_table.err; echo "rate rc $?" >> $O/rate_table.err
