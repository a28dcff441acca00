# conv2 backward-data (BN 96): CTA pairs (default) vs single CTAs with merged products (A_TMEM 3)
O=gpurun_out/r3zh; mkdir -p $O
for r in 1 2; do
for t in "" "a_tmem=3,cta_pairs=1" "cta_pairs=1" "a_tmem=2" "a_tmem=3"; do
  echo "tune [$t]: $(python tools/pass_time.py --layer conv2 --pass dgrad --layout 1 --reps 10 ${t:+--tune $t} 2>&1 | tail -1)" >> $O/pt.log
done
done
