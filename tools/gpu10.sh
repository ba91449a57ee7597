set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu10.log
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench10.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench10.log
PMAP_NO_P2REC=1 timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench10_norec.log 2>&1
