set -o pipefail
mkdir -p gpurun_out
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench12.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench12.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain12.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p1_tiles|k_p1_groups|k_p1_reduce_lti_edge|k_p1_down|k_p2_down" -s 10 -c 6 -o gpurun_out/prof12 $CMD > gpurun_out/ncu12.log 2>&1
echo "ncu rc=$?" >> gpurun_out/plain12.log
