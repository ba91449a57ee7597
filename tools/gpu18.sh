set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_next_rows_gpu.py -q -x > gpurun_out/p18_next.log 2>&1; echo "rc=$?" >> gpurun_out/p18_next.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/p18_all.log 2>&1; echo "rc=$?" >> gpurun_out/p18_all.log
for c in C2E C2 C5; do
timeout 600 python bench.py --config $c --steps 50 --no-e2e > gpurun_out/b18_$c.log 2>&1
done
