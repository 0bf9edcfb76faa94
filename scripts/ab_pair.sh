#!/bin/bash
# Dev aid: same-box A/B of the c2 LRNR and FastLRNR sweeps for the default library and
# variant libraries (scripts/liblrnr_gpu_NAME.so from scripts/build_core_variant.sh):
#   bash scripts/ab_pair.sh NAME [NAME...]   (run on the GPU box)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then lib=""; else lib="LRNR_GPU_LIB=scripts/liblrnr_gpu_$v.so"; fi
    env $lib timeout 120 python scripts/lrnr_ab.py | grep '"l2_flush": 1' | sed "s/^/$v lrnr /"
    env $lib timeout 300 python scripts/fast_ab.py | grep '"kernel": 0' | sed "s/^/$v fast /"
  done
done
