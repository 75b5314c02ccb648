#!/bin/bash
# conv_fwd shared-memory budget per CTA (2 vs 3 CTAs per SM) on C4 and C3 (gpurun box).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for B in 113 74; do
  SPC_FWD_BUDGET_KB=$B timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --sweep none --no-key32 > gpurun_out/fb_c4_$B.log 2>&1
  SPC_FWD_BUDGET_KB=$B timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config c3 > gpurun_out/fb_c3_$B.log 2>&1
done
python - <<'PY'
import json
for B in (113, 74):
    for c in ("c4", "c3"):
        try:
            d = json.loads([l for l in open(f"gpurun_out/fb_{c}_{B}.log") if l.startswith("{")][-1])
            k = d["kernels"]
            f = lambda n: (k[n]["ms"] if isinstance(k[n], dict) else k[n]) if n in k else None
            print(B, c, d["ms_per_step"], "fwd", f("conv_fwd"), "sample", f("conv_fwd_sample"))
        except Exception as e:
            print(B, c, "fail", e)
PY
