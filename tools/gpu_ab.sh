# interleaved same-box A/B of the bench step: the previous build (abtest/old, a git worktree built
# in place) against the working tree, optional tuning variants of the new build (NEWTUNES)
O=gpurun_out/${AB_TAG:-ab}; mkdir -p $O
for r in 1 2 3; do
  (cd abtest/old && timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu --no-configs) > $O/old_$r.json 2>$O/old_$r.err
  for t in ${NEWTUNES:-none}; do
    if [ "$t" = none ]; then a=""; else a="--tune $t"; fi
    timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu --no-configs $a > $O/new_${t}_$r.json 2>$O/new_${t}_$r.err
  done
done
