# A/B of the Jacobi early exit (NYS_JACOBI_VERIFY=1 = always run the verifying sweep)
for sh in "2000x8000 50" "64x200000 64" "20000x20000 100" "50000x20000 200"; do
  for v in "" 1; do
    echo "== $sh VERIFY=$v"; NYS_JACOBI_VERIFY=${v:-0} python tools/sketch_bench.py $sh 7 2>&1 | tail -2
  done
done
for c in 1 3 0; do
  for v in "" 1; do
    echo "== config $c VERIFY=$v"; NYS_JACOBI_VERIFY=${v:-0} python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d.get('solve',{}).get('outer'), d.get('solve',{}).get('inner'), d.get('solve',{}).get('obj'))"
  done
done
