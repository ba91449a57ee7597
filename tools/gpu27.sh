mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/p27_all.log 2>&1; echo "rc=$?" >> gpurun_out/p27_all.log
