#!/bin/bash
# Round-2 checkpoint captures (GPU box, repo root): GPU tests, smoke, default bench line, launch
# list, ncu --set full of the dominant kernels (each workload first exits 0 without ncu).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
T=${TAG:-v7}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_gputest_$T.txt 2>&1; tail -3 gpurun_out/r02_gputest_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_$T.txt 2>&1; tail -1 gpurun_out/r02_smoke_$T.txt
timeout 900 python bench.py > gpurun_out/r02_bench_$T.json 2> gpurun_out/r02_bench_$T.err; tail -c 400 gpurun_out/r02_bench_$T.json
for w in c3 c2; do timeout 300 python tools/ncu_work.py $w 3 > /dev/null 2>&1 || exit 1; done
cap() { timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:$1" -s $2 -c ${5:-1} -o gpurun_out/r02_$3_$T -f python tools/ncu_work.py $4 3 > gpurun_out/r02_$3_$T.log 2>&1; }
cap "k_gemm<.int.4>" 6 gemm_bwdln_c2 c2
cap "k_chain" 6 chain_c2 c2
cap "k_gemm<.int.0>" 4 gemm_ln_c3 c3
cap "k_gemm_ln16<.int.4>" 4 gemm_ln16_c3 c3
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_$T.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02_launches_$T.log 2>&1
ls -la gpurun_out/r02_*_$T*
