mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-seq"
ncu --set full --clock-control none --import-source on -k regex:"k_p1_down" -s 2 -c 1 -o gpurun_out/p34_prof $CMD > gpurun_out/p34_ncu.log 2>&1
