#!/bin/bash
# FAST v2 occupancy x burst A/B
export PYTHONPATH=$PWD
O=gpurun_out
bash tools/ab_variants.sh fast v1 c6 c6b32 c6b64 c5b32 c5b64 c6b32f8 c6b32r8 v1 > $O/ab_x.txt 2>&1
