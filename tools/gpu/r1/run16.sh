mkdir -p gpurun_out/ds
for L in paper_1906_06504_b200/libbatchheap_b200.so exp/lib_lf.so; do
  echo "== $L"
  BH_LIB=$PWD/$L timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 --profile 2>&1 | grep -E "k=|serving"
  BH_LIB=$PWD/$L timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 2>&1 | grep -E "k="
done > gpurun_out/ds/exp16.log 2>&1
cat gpurun_out/ds/exp16.log
