#!/bin/bash
# usage: tools/variant_bench_cfg.sh CONFIG v1 v2 ...   (tools/variants/<v>.so swapped in, bench.py --config CONFIG)
cfg=$1; shift
cp paper_1702_07578_b200/_wvlt_b200.so /tmp/_orig.so
for v in "$@"; do
  cp tools/variants/$v.so paper_1702_07578_b200/_wvlt_b200.so
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-wt --config $cfg > gpurun_out/var_${cfg}_$v.json 2> gpurun_out/var_${cfg}_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/var_${cfg}_$v.json')); print('$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
cp /tmp/_orig.so paper_1702_07578_b200/_wvlt_b200.so
