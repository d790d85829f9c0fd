#!/bin/bash
# Time the fused decode linear with parts of it disabled (ARC_FUSED_DEBUG bits, timing only).
for d in ${@:-0 16 4 15}; do
  echo "== ARC_FUSED_DEBUG=$d"
  ARC_FUSED_DEBUG=$d timeout 120 python scripts/time_decode.py fused 2>&1 | grep -E "M=  1|M= 16|M=128"
done
