# interleaved same-box A/B of the bench step: the previous build (abtest/old, a git worktree built
# in place) against the working tree, tuning variants of the new build (NEWTUNES) and compile-time
# variants (VARIANTS: abtest/NAME/libcct.so from tools/build_variant.sh, loaded with CCT_LIB_DIR)
O=gpurun_out/${AB_TAG:-ab}; mkdir -p $O
B="--steps 30 --warmup 5 --no-e2e --no-cpu --no-configs"
for r in 1 2 3; do
  [ -d abtest/old ] && (cd abtest/old && timeout 300 python bench.py $B) > $O/old_$r.json 2>$O/old_$r.err
  for t in ${NEWTUNES:-none}; do
    if [ "$t" = none ]; then a=""; else a="--tune $t"; fi
    timeout 300 python bench.py $B $a > $O/new_${t}_$r.json 2>$O/new_${t}_$r.err
  done
  for v in ${VARIANTS:-}; do
    CCT_LIB_DIR=abtest/$v timeout 300 python bench.py $B > $O/var_${v}_$r.json 2>$O/var_${v}_$r.err
  done
done
