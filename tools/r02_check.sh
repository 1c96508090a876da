#!/bin/bash
# gpu tests + parity bench + ncu of the parity tracer (round-2 iteration check)
export PYTHONPATH=$PWD
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --mode parity --no-extras --no-cpu-baseline --steps 20 > $O/bench_parity.json 2> $O/bench_parity.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_render_trace" -s 1 -c 1 \
    -o $O/trace_parity python tools/profile_frame.py --mode parity --frames 2 > $O/ncu_parity.log 2>&1
python tools/ncu_summary.py $O/trace_parity.ncu-rep $O/trace_parity_sum > /dev/null 2>&1
