set -o pipefail
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-seq"
$CMD > gpurun_out/p19_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_p1_reduce_lti|k_p1_tiles|k_p1_groups|k_p2_tiles|k_p2_groups" -s 14 -c 6 -o gpurun_out/p19_prof $CMD > gpurun_out/p19_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p19_ncu.log
