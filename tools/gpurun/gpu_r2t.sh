# round-2 call T: fused Types 2/3 tests + full GPU suite + smoke
O=gpurun_out/r2t; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "fused_types or implicit" -q --timeout 500 > $O/fused.log 2>&1; echo "fused rc $?" >> $O/fused.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
