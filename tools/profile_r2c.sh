#!/bin/bash
# Round-2 final captures (run on the GPU box from the repo root; each workload exits 0 first).
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for w in c3 c2; do timeout 300 python tools/ncu_work.py $w 3 || exit 1; done
cap() { timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:$1" -s $2 -c ${5:-1} -o gpurun_out/r02_$3 -f python tools/ncu_work.py $4 3 > gpurun_out/r02_$3.log 2>&1; }
cap "k_gemm_ln16<.int.4>" 4 gemm_ln16_c3 c3 2
cap "k_enc_bwd_tc<.int.64>" 1 enc_bwd_c3 c3
cap "k_enc_fwd_ws<.int.64>" 1 enc_fwd_c3 c3
cap "k_chain" 6 chain_c2 c2
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02_launches_bench.log 2>&1
ls -la gpurun_out/r02_*
