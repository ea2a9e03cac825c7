# Same-box A/B of library builds (profiles/r2/ab_final.txt): bench.py without
# extras under each library (BH_LIB), libraries interleaved, REPS rounds.
# Build a variant with a patched copy of the tree, e.g.
#   git worktree add --detach build_var/wt_X HEAD   (patch its csrc)
#   make -C build_var/wt_X/paper_1906_06504_b200/csrc DEV=1 -j8
#   cp build_var/wt_X/paper_1906_06504_b200/libbatchheap_b200.so build_var/lib_X.so
# then: LIBS="base X" REPS="1 2 3" bash tools/gpu/ab.sh   (under gpurun)
OUT=gpurun_out/ab; mkdir -p $OUT
for rep in ${REPS:-1 2}; do
  for lib in ${LIBS:?set LIBS to build_var/lib_<name>.so names}; do
    BH_LIB=build_var/lib_$lib.so timeout 600 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 5 --warmup 3 \
      > $OUT/$lib.$rep.json 2> $OUT/$lib.$rep.err
    python -c "
import json; d=json.loads(open('$OUT/$lib.$rep.json').read().strip().splitlines()[-1])
print('$lib rep $rep', round(d['value']/1e6,1), 'ins', d['insert_ms_stats'], 'del', round(d['delete_ms'],1), d['clocks']['sm_mhz'])"
  done
done
