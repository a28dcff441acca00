# lift / expand kernels of the configs[1] sweep: ncu --set full (T3 and T2, d = o = 256, b = 256)
O=gpurun_out/r3t; mkdir -p $O; R=/tmp/reps; mkdir -p $R
for t in 3 2; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"lift|expand" -o $R/le$t -f \
      python tools/layer_step.py 13 3 256 256 1 1 $t > $O/ncu_$t.log 2>&1
  python tools/ncu_summary.py $R/le$t.ncu-rep "T$t lift / expand (n 13, k 3, d = o = 256, b 256)" > $O/le$t.txt
  ncu -i $R/le$t.ncu-rep --page raw --csv > $O/le${t}_raw.csv 2>/dev/null
done
