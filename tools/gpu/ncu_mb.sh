set -x
mkdir -p gpurun_out
for v in m0 m8 m3; do
  ncu --set full --import-source on -k regex:merge_bench -c 1 -o gpurun_out/mb_$v -f tools/microbench/mb $v > gpurun_out/mb_$v.log 2>&1
done
ls -la gpurun_out
