set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 900 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench4.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_p1_reduce_lti|k_p1_down" -s 2 -c 3 -o gpurun_out/prof_r01b $CMD > gpurun_out/ncu4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/plain4.log
