#!/bin/bash
# A/B of the in-tree library against tools/libddppo_old.so on one bench config, alternating runs.
# usage: tools/ab.sh CONFIG STEPS ROUNDS
cfg=${1:-depth}; steps=${2:-10}; rounds=${3:-2}
cp paper_1911_00357_b200/libddppo.so /tmp/new.so
for i in $(seq $rounds); do
  for v in new old; do
    if [ $v = old ]; then cp tools/libddppo_old.so paper_1911_00357_b200/libddppo.so; else cp /tmp/new.so paper_1911_00357_b200/libddppo.so; fi
    python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > /tmp/ab.json
    python -c "import json;d=json.load(open('/tmp/ab.json'));print('$v',round(d['value']),round(d['ms_per_step'],3),{k:round(v/d['kernel_ms_steps'],2) for k,v in d['kernel_ms'].items()})"
  done
done
cp /tmp/new.so paper_1911_00357_b200/libddppo.so
