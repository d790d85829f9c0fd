#!/bin/bash
# Time arc_gemm (isolated, CUDA graph) for the LLaMA-3-8B sites under env-selected kernel variants.
# usage: bash scripts/gemm_variants.sh [--M m] "VAR=.. VAR2=.." "..." ...   (one process per variant)
cd "$(dirname "$0")/.."
M=8192
if [ "$1" == "--M" ]; then M=$2; shift 2; fi
for v in "$@"; do
  env $v python scripts/time_gemm.py --M $M 2>&1 | grep -E "TFLOP|Error|error" 
done
