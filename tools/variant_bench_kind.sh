#!/bin/bash
# usage: tools/variant_bench_kind.sh CONFIG KIND v1 v2 ...   (tools/variants/<v>.so swapped in, bench.py --config CONFIG --kind KIND)
cfg=$1; kind=$2; shift 2
cp paper_1702_07578_b200/_wvlt_b200.so /tmp/_orig.so
for v in "$@"; do
  cp tools/variants/$v.so paper_1702_07578_b200/_wvlt_b200.so
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-wt --config $cfg --kind $kind > gpurun_out/var_${cfg}_${kind}_$v.json 2> gpurun_out/var_${cfg}_${kind}_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/var_${cfg}_${kind}_$v.json')); print('$cfg $kind $v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
cp /tmp/_orig.so paper_1702_07578_b200/_wvlt_b200.so
