set -o pipefail
mkdir -p gpurun_out
for c in C4 C5 C2; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench7_$c.log 2>&1
done
