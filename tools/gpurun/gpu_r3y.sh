O=gpurun_out/r3y; mkdir -p $O; R=/tmp/reps; mkdir -p $R
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"expand" -o $R/ex3 -f \
    python tools/layer_step.py 13 3 256 256 1 1 3 > $O/ncu_3.log 2>&1
ncu -i $R/ex3.ncu-rep --page raw --csv > $O/ex3_raw.csv 2>/dev/null
ncu -i $R/ex3.ncu-rep --page source --csv --print-source sass > $O/ex3_sass.csv 2>/dev/null
ls -la $O
