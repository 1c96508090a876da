#!/bin/bash
# Round-2 first GPU pass: gpu tests, bench (fast + parity), ncu of the parity tracer.
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --mode parity --no-extras --no-cpu-baseline > $O/bench_parity.json 2> $O/bench_parity.err
timeout 300 python bench.py --mode fast --no-extras --no-cpu-baseline > $O/bench_fast.json 2> $O/bench_fast.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_render_trace" -s 1 -c 1 \
    -o $O/trace_parity python tools/profile_frame.py --mode parity --frames 2 > $O/ncu_parity.log 2>&1
python tools/ncu_summary.py $O/trace_parity.ncu-rep $O/trace_parity_sum > /dev/null 2>&1
python tools/ncu_hotspots.py $O/trace_parity.ncu-rep k_render_trace 40 > $O/hot_trace_parity.md 2>&1
ls -la $O
