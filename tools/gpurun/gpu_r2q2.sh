# round-2 call Q2: smoke (with the fused conv1 case) + full GPU suite on the current build
O=gpurun_out/r2q2; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
