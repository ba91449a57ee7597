set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
timeout 900 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/bench3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench3.log
PMAP_GENERAL=1 timeout 900 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bench3_general.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench3_general.log
