#!/bin/bash
# K3 regime sweep over env knob settings: VARIANTS="A=1,B=2 A=0" SPECS="c1:0.95 ..."
mkdir -p gpurun_out
i=0
for v in ${VARIANTS:-none}; do
  i=$((i+1))
  envs=$(echo "$v" | tr ',' ' '); [ "$v" = none ] && envs=""
  env $envs timeout 300 python tools/k3_regimes.py $SPECS > gpurun_out/k3reg_$i.log 2>&1
  echo "== $v rc=$?"
  python - "$i" <<'PY'
import json, sys
for l in open(f"gpurun_out/k3reg_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l); t = d["traced_step"]
        print(d["workload"], d["T"], round(d["k3_us_per_step"], 2), round(d["frac_of_measured_peak"], 3),
              "iso", t["isolated_step_us"], "plan", t["plan_us_median"], "first", t["first_page_us_median"],
              "lastpg", t["last_page_us_median"], "tail", [round(x, 1) for x in t["tail_after_last_page_us"]],
              "phases", t.get("phase_cycles_median"))
    elif "Error" in l or "error" in l:
        print(l.strip()[:300])
PY
done
