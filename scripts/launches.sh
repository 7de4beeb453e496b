#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in ${CFGS:-c2 c5}; do
timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_${c}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file gpurun_out/${TAG}_${c}_launches.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo "$c=$?"
python - "$TAG" "$c" <<'PY'
import csv, sys
tag, c = sys.argv[1], sys.argv[2]
rows=[r for r in csv.reader(l for l in open(f"gpurun_out/{tag}_{c}_launches.csv") if not l.startswith("=="))]
h=rows[0]; ks={}
order=[]
for r in rows[1:]:
    d=dict(zip(h,r)); key=(d['ID'], d['Kernel Name'][:30])
    if key not in ks: ks[key]={}; order.append(key)
    ks[key][d['Metric Name']]=d['Metric Value']
out=[]
for key in order[:16]:
    m=ks[key]
    out.append(f"{key[1][6:20]} {float(m.get('gpu__time_duration.sum',0))/1e3:.1f}us iss{float(m.get('smsp__issue_active.avg.pct_of_peak_sustained_active',0)):.0f} wa{float(m.get('sm__warps_active.avg.pct_of_peak_sustained_active',0)):.0f}")
print(c, " | ".join(out))
PY
done
