set -o pipefail
mkdir -p gpurun_out
#timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu5.log
for v in main b6 b8; do
  if [ "$v" = main ]; then L=""; else L="$PWD/variants/libpmap_$v.so"; fi
  PMAP_LIB=$L timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench5_$v.log 2>&1
done
