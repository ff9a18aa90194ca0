# A/B: default kernels vs SB200_NO_PIPE / SB200_NO_TMA fallbacks (bench, no e2e / cpu legs)
set -x
R=${1:-ab}
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${R}_new.json 2>&1
SB200_NO_PIPE=1 SB200_NO_TMA=1 timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${R}_old.json 2>&1
python - <<PY
import json
for tag in ("new","old"):
    j=json.load(open(f"gpurun_out/ab_${R}_{tag}.json"))
    print(tag, j["value"], {k:v["GBps"] for k,v in j["per_test"].items()})
PY
