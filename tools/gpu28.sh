mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/p28_all.log 2>&1; echo "rc=$?" >> gpurun_out/p28_all.log
for c in C3 C4 C2; do timeout 600 python bench.py --config $c --steps 100 --no-cpu-baseline --no-e2e --no-seq > gpurun_out/b28_$c.log 2>&1; done
for G in 8; do timeout 300 python tools/shard_probe.py $G >> gpurun_out/p28_probe.log 2>&1; done
