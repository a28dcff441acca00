# round-2 call J: row-stage waits spin instead of sleep (A/B vs call I)
O=gpurun_out/r2j; mkdir -p $O
timeout 120 python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass wgrad --layout 1 --reps 20 >> $O/time.log 2>&1
timeout 120 python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 20 >> $O/time.log 2>&1
