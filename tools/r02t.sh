#!/bin/bash
# field encoder levels-per-sweep / occupancy A/B + PARITY refill threshold A/B
export PYTHONPATH=$PWD
O=gpurun_out
bash tools/ab_variants.sh parity default g2 g8 m6 m8 r1 r2 r3 default > $O/ab_t.txt 2>&1
