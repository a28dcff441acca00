# round-2 call L2: full GPU suite after the CH2 MN/MN fix
O=gpurun_out/r2l2; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/tests.log 2>&1; echo "tests rc $?" >> $O/tests.log
