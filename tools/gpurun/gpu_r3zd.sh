# e2e copy-path variants on one box
O=gpurun_out/r3zd; mkdir -p $O
for r in 1 2; do
  for v in "--copy-streams 1" "--copy-streams 2" "--copy-streams 3" "--copy-streams 1 --h2d-wc 1" "--copy-streams 2 --h2d-wc 1"; do
    n=$(echo $v | tr -d ' -'); timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-configs $v > $O/e2e_${n}_$r.json 2>$O/e2e_${n}_$r.err
  done
done
