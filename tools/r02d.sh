#!/bin/bash
# field lane-pair encoder + parity step trims: targeted tests, bench line, ncu of the field kernels + parity tracer
export PYTHONPATH=$PWD
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_c2.py tests/test_gpu_tracking.py tests/test_golden.py tests/test_gpu_render.py tests/test_gpu_train.py -m gpu -q -x > $O/pytest_d.log 2>&1; echo "rc=$?" >> $O/pytest_d.log
timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 > $O/bench_d.json 2> $O/bench_d.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_field|k_render_trace_parity" -s 3 -c 3 \
    -o $O/frame_d python tools/profile_frame.py --mode parity --frames 2 > $O/ncu_d.log 2>&1
python tools/ncu_summary.py $O/frame_d.ncu-rep $O/frame_d_sum > /dev/null 2>&1
ls -la $O
