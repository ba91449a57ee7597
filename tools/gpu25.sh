mkdir -p gpurun_out
timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b25_mb8s4.log 2>&1
for v in mb12s4; do
PMAP_LIB=variants/$v/libpmap.so timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b25_$v.log 2>&1
done
