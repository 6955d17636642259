#!/bin/bash
# Round-2 follow-up captures (run on the GPU box from the repo root after the workloads exit 0):
# the c4 act's pipelined squint + encoder (k_enc_fwd_ws<32>) and the c3 LayerNorm GEMMs.
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for w in c3; do timeout 300 python tools/ncu_work.py $w 3 || exit 1; done
cap() { timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:$1" -s $2 -c ${5:-1} -o gpurun_out/r02_$3 -f python tools/ncu_work.py $4 3 > gpurun_out/r02_$3.log 2>&1; }

cap "k_gemm<.int.4>" 6 gemm_bwdln_c3 c3 2
cap "k_gemm<.int.0>" 4 gemm_ln_c3 c3 2
ls -la gpurun_out/r02_*
