#!/bin/bash
# Profiling recipe (run under gpurun, 1 GPU).  Outputs land in gpurun_out/.
#  1. launch list of a 2-layer C2 step (every kernel, device time; cold-cache, serialised)
#  2. one `ncu --set full` capture of the sparse attention kernel (layer 0 of C2)
set -x
OUT=gpurun_out
ARGS="--layers 2 --steps 1 --warmup 3 --no-cpu --no-e2e --no-dense"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py $ARGS > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_fwd -s 3 -c 1 \
    -o $OUT/attn_full -f python bench.py --layers 1 --steps 1 --warmup 3 --no-cpu --no-e2e --no-dense \
    > $OUT/attn_full.log 2>&1
ls -la $OUT
