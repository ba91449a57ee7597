set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "c3_full" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c3.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/plain.log
ncu --set full --clock-control none --import-source on -k regex:"k_p1_reduce|k_p1_down|k_p2_down" -s 3 -c 3 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/plain.log
