#!/bin/bash
# A/B of libpfgpu variants (tools/build_variant.py) on the C2 bench; args: mode variant...
# Tooling, not product.  Output: gpurun_out/ab_<mode>_<variant>.json
export PYTHONPATH=$PWD
mode=$1; shift
for v in "$@"; do
  if [ $v = default ]; then unset PF_LIBPFGPU; else export PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_$v.so; fi
  timeout 300 python bench.py --mode $mode --no-extras --no-cpu-baseline --steps 20 > gpurun_out/ab_${mode}_$v.json 2> gpurun_out/ab_${mode}_$v.err
done
unset PF_LIBPFGPU
for v in "$@"; do python - "$mode" "$v" <<'PY'
import json, sys
m, v = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{m}_{v}.json").read().strip().splitlines()[-1])
    f = d["frame"]
    print(f"{v:10s} fps {d['value']:8.2f} trace {f['ms_trace']:.3f} field {f['ms_field']:.3f} hits {f['hits']:.0f} steps/sample {f['steps_per_sample']:.4f}")
except Exception as e:
    print(v, "failed", e)
PY
done
