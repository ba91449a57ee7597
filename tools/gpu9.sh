set -o pipefail
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain9.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_p1_reduce_lti<|k_p1_tiles|k_p1_groups" -s 3 -c 3 -o gpurun_out/prof9 $CMD > gpurun_out/ncu9.log 2>&1
echo "ncu rc=$?" >> gpurun_out/plain9.log
