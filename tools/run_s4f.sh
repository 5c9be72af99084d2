# weight-spectrum cache: ncu launch list of the pre-pass kernels (16 frames, fp64), configs 1/2/3/5 on/off
set -x
mkdir -p gpurun_out
T=${TAG:-s4f}
P="python tools/prof_run.py --frames 16 --precision fp64 --reps 2"
$P > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_wc1.csv $P > gpurun_out/${T}_ncu_wc1.log 2>&1
python - <<'PY'
import csv, collections, os, re
T=os.environ.get("TAG","s4f")
f=f"gpurun_out/{T}_launches_wc1.csv"
rows=[r for r in csv.reader(open(f, errors="replace")) if len(r)>5]
hdr=None; agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if not hdr: continue
    d=dict(zip(hdr,r))
    if d.get("Metric Name")!="gpu__time_duration.sum": continue
    name=re.sub(r"\(.*","",d["Kernel Name"])[:110]
    v=float(d["Metric Value"].replace(",","")); u=d["Metric Unit"]
    v*= {"ns":1e-6,"us":1e-3,"usecond":1e-3,"nsecond":1e-6,"msecond":1,"ms":1}.get(u,1e-6)
    agg[name][0]+=1; agg[name][1]+=v
for k,(n,ms) in sorted(agg.items(), key=lambda x:-x[1][1])[:12]:
    print(f"   {ms:10.3f} ms {n:6d}  {k}")
PY
for wc in ; do
  for c in 1 2; do FSE_WCACHE=$wc python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c${c}_wc$wc.json 2>&1; done
  FSE_WCACHE=$wc python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c3_wc$wc.json 2>&1
  for B in 2 4 8; do FSE_WCACHE=$wc python bench.py --config 5 --block $B --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-second > gpurun_out/${T}_c5b${B}_wc$wc.json 2>&1; done
done
python - <<'PY'
import json,glob,os
T=os.environ.get("TAG","s4f")
for f in sorted(glob.glob(f"gpurun_out/{T}_c*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["dtype"], round(d["ms_per_step"],2), round(d["kernel_ms_per_step"],2), (d.get("weight_spectrum_cache") or {}).get("hit_share"), (d.get("weight_spectrum_cache") or {}).get("planes_per_step"))
    except Exception as e:
        print(f, "ERR", e); print(open(f).read()[-800:])
PY
