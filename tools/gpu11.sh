set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu11.log
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench11.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench11.log
timeout 600 python bench.py --config C5 --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench11_c5.log 2>&1
