set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final_bench.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/final_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/final_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_p1_down|k_p2_down|k_p1_reduce_lti|k_p1_tiles|k_p1_groups" -s 8 -c 5 -o gpurun_out/final_prof $CMD > gpurun_out/final_ncu2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/final_plain.log
