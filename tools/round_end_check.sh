#!/bin/bash
# What the driver runs on the GPU box at round end, in order (one GPU):
# GPU tests, smoke(), the reference arm, then our bench.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/rc_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/rc_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference > $OUT/rc_ref.json 2> $OUT/rc_ref.err; echo "reference arm rc=$?"
timeout 900 python bench.py > $OUT/rc_bench.json 2> $OUT/rc_bench.err; echo "bench rc=$?"
tail -1 $OUT/rc_gpu_tests.log; tail -1 $OUT/rc_smoke.log
python - <<'PY'
import json
for f in ("gpurun_out/rc_ref.json", "gpurun_out/rc_bench.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("impl", "ours"), d["value"], d["unit"], "e2e", d["e2e"]["value"])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
PY
