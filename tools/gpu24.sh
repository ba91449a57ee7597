mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/p24_all.log 2>&1; echo "rc=$?" >> gpurun_out/p24_all.log
timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b24.log 2>&1
