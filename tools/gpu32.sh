mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-seq"
ncu --set full --clock-control none --import-source on -k regex:"k_p1_tiles_lti|k_p1_groups_lti" -s 2 -c 2 -o gpurun_out/p32_prof $CMD > gpurun_out/p32_ncu.log 2>&1
