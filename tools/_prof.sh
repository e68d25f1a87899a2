#!/bin/bash
# one ncu --set full capture of the byte pass (c2) for the product library [+ a variant]
set -u
TAG=${TAG:-q}
python tools/run_build.py --config ${CFG:-c2} --iters 1 > gpurun_out/rb.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"${KRE:-level_pass8}" -c 1 -o gpurun_out/${TAG}full python tools/run_build.py --config ${CFG:-c2} --iters 1 > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
