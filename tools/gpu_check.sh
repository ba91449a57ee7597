# Quick GPU check: all GPU tests, C3/C2/C5 bench lines without baselines, the 8-way shard probe.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/p33_all.log 2>&1; echo "rc=$?" >> gpurun_out/p33_all.log
for c in C3 C2 C5; do timeout 600 python bench.py --config $c --steps 100 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b33_$c.log 2>&1; done
for G in 8; do timeout 300 python tools/shard_probe.py $G >> gpurun_out/p33_probe.log 2>&1; done
