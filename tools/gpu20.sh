set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_next_rows_gpu.py -q -x -k "mask" > gpurun_out/p20_mask.log 2>&1; echo "rc=$?" >> gpurun_out/p20_mask.log
timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b20_C3.log 2>&1
PMAP_NO_MASK=1 timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b20_C3_nomask.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/p20_all.log 2>&1; echo "rc=$?" >> gpurun_out/p20_all.log
