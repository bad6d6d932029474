#!/bin/bash
# Runs bench.py over a list of argument sets (one per line of $SWEEP), logs to gpurun_out/sweep_*.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
i=0
while IFS= read -r args; do
  [ -z "$args" ] && continue
  i=$((i+1))
  timeout ${ONE_TIMEOUT:-600} python bench.py $args > gpurun_out/sweep_$i.json 2> gpurun_out/sweep_$i.log
  echo "== [$i] $args rc=$?"
  grep -E "swap batch|OOM at|no-swap" gpurun_out/sweep_$i.log | tail -4
  python - "$i" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/sweep_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    s = d["swap"]
    print(" value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"], "batch", d["config"]["per_gpu_batch"],
          "n_t", s["tensors_swapped"], "d2hGB", round(s["d2h_bytes_per_step"]/1e9, 2), "h2dGB", round(s["h2d_bytes_per_step"]/1e9, 2),
          "d2h_rate", s["d2h_gbs_while_busy"], "h2d_rate", s["h2d_gbs_while_busy"], "wait_ms", s["swap_wait_ms_per_step"],
          "launches", d["gpu_launches"])
except Exception as e:
    print(" no json", e)
PY
done <<< "$SWEEP"
