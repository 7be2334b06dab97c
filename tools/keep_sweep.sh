for cfg in 1 3; do
for pf in d 0; do
for keep in 0 4 6 8 10 12 16 100; do
  if [ $pf = d ]; then unset NYS_PCG_PF; else export NYS_PCG_PF=$pf; fi
  echo "cfg $cfg pf $pf keep $keep: $(NYS_PCG_KEEP=$keep python tools/pcg_fixed.py $cfg 400 2>&1 | tail -1)"
done; done; done
