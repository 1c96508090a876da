#!/bin/bash
# PARITY pipelined tracer: refill threshold / burst length A/B
export PYTHONPATH=$PWD
O=gpurun_out
bash tools/ab_variants.sh parity default r2 r8 b12 b20 default > $O/ab_s.txt 2>&1
