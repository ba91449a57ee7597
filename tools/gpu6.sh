set -o pipefail
mkdir -p gpurun_out
for c in C1 C2 C4 C5; do
  timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench6_$c.log 2>&1
done
