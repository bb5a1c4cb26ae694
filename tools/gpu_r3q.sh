# fcgscan variants: main (g^ in TMEM, row-mapped C, 4 stages), s3 (same, 3 stages), head, alias (timing only)
for v in main s3 head alias; do
  if [ $v = main ]; then unset TERN_LIB; else export TERN_LIB=$PWD/build/var_$v/libtern.so; fi
  for c in c2 c3 c4; do echo "$v $c $(timeout 300 python tools/kernel_breakdown.py --config $c --prefill --blocks 2 2>&1 | grep -i fcg)"; done
done
