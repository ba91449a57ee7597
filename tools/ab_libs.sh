#!/bin/bash
# A/B of several builds of libpmap.so on the default bench line: ab_libs.sh lib1.so lib2.so ...
# (each lib under paper_2512_13319_b200/; env vars in AB_ENV apply to every run)
for rep in 1 2; do
  for L in "$@"; do
    echo -n "$L rep$rep: "
    env $AB_ENV PMAP_LIB=paper_2512_13319_b200/$L timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e \
      --no-seq 2>/dev/null | head -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items()})"
  done
done
