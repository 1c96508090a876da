#!/bin/bash
# gpu tests (c2 + tracking first) + the full bench.py line + the reference arm (short)
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_tracking.py -m gpu -q -s > $O/pytest_c2.log 2>&1; echo "rc=$?" >> $O/pytest_c2.log
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
nproc > $O/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $O/nproc.txt
