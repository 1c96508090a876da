#!/bin/bash
# KNN probe growth (linear to 4, then doubling) + PARITY tracer (pipelined, 5 CTAs, fetch 2): tests, matrix, ncu
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_knn.py tests/test_gpu_tracking.py tests/test_gpu_c2.py tests/test_golden.py -m gpu -q -x > $O/pytest_n.log 2>&1; echo "rc=$?" >> $O/pytest_n.log
timeout 900 python tools/bench_knn.py > $O/knn_matrix_n.json 2> $O/knn_matrix_n.err
python tools/frame_hash.py parity > $O/hash_n.txt 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 20 > $O/bench_n.json 2> $O/bench_n.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_render_trace_parity" -s 1 -c 1 \
    -o $O/trace_parity_n python tools/profile_frame.py --mode parity --frames 2 > $O/ncu_n.log 2>&1
ncu -i $O/trace_parity_n.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_render_trace_parity > $O/trace_parity_n_src.csv 2>/dev/null
python tools/ncu_summary.py $O/trace_parity_n.ncu-rep $O/trace_parity_n_sum > /dev/null 2>&1
