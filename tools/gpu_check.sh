# Quick GPU check: all GPU tests, the default bench line and the other configs (no baselines).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/chk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/chk_pytest.log
timeout 600 python bench.py > gpurun_out/chk_bench.log 2>&1; echo "rc=$?" >> gpurun_out/chk_bench.log
for c in C1 C2 C4 C5 C2E; do timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/chk_bench_$c.log 2>&1; done
