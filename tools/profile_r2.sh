#!/bin/bash
# Round-2 profiling pass (run on the GPU box from the repo root; every run exits 0 first without ncu).
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for w in c1 c4 c3 c2; do timeout 300 python tools/ncu_work.py $w 3 || exit 1; done
# launch list of the bench step (graph replays; per-launch times cold-cache and serialised)
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02_launches_bench.log 2>&1
# one --set full capture per kernel of interest, steady-state launch
cap() { timeout 900 $NCU --set full --clock-control none --import-source on -k "regex:$1" -s $2 -c ${5:-1} -o gpurun_out/r02_$3 -f \
  python tools/ncu_work.py $4 3 > gpurun_out/r02_$3.log 2>&1; }
cap k_insert_f8 2 insert_c1 c1
cap k_enc_fwd_tc 2 act_enc_c4 c4
cap k_enc_fwd_ws 2 enc_fwd_c3 c3
cap k_enc_bwd_tc 2 enc_bwd_c3 c3
cap "k_gemm" 22 gemm_c2 c2 22
cap k_chain 6 chain_c2 c2
ls -la gpurun_out/r02_*
