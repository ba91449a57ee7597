set -o pipefail
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain13.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p1_reduce_lti$|k_p1_reduce_lti<|k_p2_tiles|k_p2_groups" -s 4 -c 3 -o gpurun_out/prof13 $CMD > gpurun_out/ncu13.log 2>&1
echo "ncu rc=$?" >> gpurun_out/plain13.log
