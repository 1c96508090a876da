#!/bin/bash
# encoder occupancy x levels-per-sweep A/B; K7c early-exit radix select: KNN tests + training bench
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_knn.py tests/test_gpu_field.py tests/test_gpu_train.py -m gpu -q -x > $O/pytest_u.log 2>&1; echo "rc=$?" >> $O/pytest_u.log
bash tools/ab_variants.sh parity default m6 m7 g4m6 default > $O/ab_u.txt 2>&1
timeout 600 python tools/bench_train.py > $O/train_u.json 2> $O/train_u.err
