#!/bin/bash
# One round's ncu evidence (run on the GPU box): the bench step's launch list (per-launch time + DRAM
# bytes), one full-set capture of the GEMM per LLaMA-3-8B site and of the quantize kernel at K=4096 /
# 14336 (M=8192), and the decode stream-K kernel.  Writes gpurun_out/<tag>_*.
tag=${1:-r2}
cd "$(dirname "$0")/.."
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    --no-streaming > gpurun_out/${tag}_launches_bench.log 2>&1
for site in qkv o gate_up down; do
  ncu --set full --clock-control none --import-source on -k regex:arc_gemm_kernel -s 1 -c 1 \
      -o gpurun_out/${tag}_gemm_${site} python scripts/prof_site.py --site $site --iters 2 > /dev/null 2>&1
done
for site in qkv down; do
  ncu --set full --clock-control none --import-source on -k regex:arc_quant_kernel -s 2 -c 1 \
      -o gpurun_out/${tag}_quant_${site} python scripts/prof_site.py --site $site --iters 2 > /dev/null 2>&1
done
ncu --set full --clock-control none -k regex:arc_gemm_kernel -s 4 -c 1 -o gpurun_out/${tag}_decode_gemm_down \
    python scripts/decode_once.py 16 down > /dev/null 2>&1
ls -la gpurun_out/ | grep ${tag}_
