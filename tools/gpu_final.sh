# Round-end evidence: GPU tests, smoke, the default bench line (+ reference arm), the
# other configs, the shard probe, the ncu launch list and one --set full capture.
set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final_bench.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1
for c in C1 C2 C4 C5 C2E; do timeout 600 python bench.py --config $c --steps 50 --no-e2e > gpurun_out/final_bench_$c.log 2>&1; done
timeout 600 python bench.py --mixed --steps 100 --no-e2e --no-cpu-baseline --no-seq > gpurun_out/final_bench_C3_mixed.log 2>&1
for G in 8 4 2; do timeout 300 python tools/shard_probe.py $G >> gpurun_out/final_shard_probe.log 2>&1; done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-seq"
$CMD > gpurun_out/final_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/final_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_lb_pass" -s 9 -c 3 -o gpurun_out/final_prof $CMD > gpurun_out/final_ncu2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/final_plain.log
