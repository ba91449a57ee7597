set -o pipefail
mkdir -p gpurun_out
for v in mb7 mb8; do
PMAP_LIB=variants/$v/libpmap.so timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench16_$v.log 2>&1
done
