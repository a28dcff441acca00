O=gpurun_out/r3s; mkdir -p $O
./tools/gather_probe 256 > $O/gprobe.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_fwd_gather --csv --log-file $O/ncu_pace.csv ./tools/gather_probe 256 > $O/gprobe_ncu.log 2>&1
