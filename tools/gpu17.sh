set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_next_rows_gpu.py -q -x > gpurun_out/p17_next.log 2>&1; echo "rc=$?" >> gpurun_out/p17_next.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/p17_all.log 2>&1; echo "rc=$?" >> gpurun_out/p17_all.log
for c in C2 C4 C5 C1; do
timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/b17_$c.log 2>&1
done
timeout 900 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/b17_C3.log 2>&1
