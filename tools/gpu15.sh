set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu15.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu15.log
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench15.log 2>&1
for v in mb7 mb8; do
PMAP_LIB=variants/$v/libpmap.so timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench15_$v.log 2>&1
done
