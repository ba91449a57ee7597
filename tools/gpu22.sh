mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "shard or nccl or both_run or filter" > gpurun_out/p22_shard.log 2>&1; echo "rc=$?" >> gpurun_out/p22_shard.log
for G in 8 2; do timeout 300 python tools/shard_probe.py $G >> gpurun_out/p22_probe.log 2>&1; done
