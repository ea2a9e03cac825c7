# strict ins-del pairs at full size under each library build (BH_LIB), 90 s each
for lib in ${LIBS:-build_var/lib_varA.so}; do
  for f in 0x0; do
    echo "== $lib flags=$f"
    BH_LIB=$lib timeout 90 python tools/probe_mixed.py --variants bu --reps 1 --flags $f 2>&1 | tail -1
  done
done
