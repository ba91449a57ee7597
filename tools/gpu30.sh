mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-seq"
$CMD > gpurun_out/p30_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_p1_down|k_p2_down|k_p1_reduce_lti" -s 6 -c 4 -o gpurun_out/p30_prof $CMD > gpurun_out/p30_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p30_ncu.log
