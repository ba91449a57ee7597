mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b21_C3.log 2>&1
for G in 8 4 2; do timeout 300 python tools/shard_probe.py $G >> gpurun_out/p21_shard.log 2>&1; done
