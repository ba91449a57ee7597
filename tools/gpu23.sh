mkdir -p gpurun_out
timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b23_base.log 2>&1
PMAP_LIB=variants/mb12/libpmap.so timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b23_mb12.log 2>&1
