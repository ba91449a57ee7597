set -o pipefail
mkdir -p gpurun_out
for v in main nospec spec_u2; do
  if [ "$v" = main ]; then L=""; else L="$PWD/variants/libpmap_$v.so"; fi; PMAP_LIB=$L timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench8_$v.log 2>&1
done
