# weight-spectrum cache diagnostics: ncu launch lists (16 frames, fp64) with the cache on / off
set -x
mkdir -p gpurun_out
T=${TAG:-s4b}
P="python tools/prof_run.py --frames 16 --precision fp64 --reps 2"
for wc in 0 1; do
  FSE_WCACHE=$wc $P > /dev/null 2>&1 && \
  FSE_WCACHE=$wc ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_wc$wc.csv $P > gpurun_out/${T}_ncu_wc$wc.log 2>&1
done
FSE_WCACHE=1 FSE_WCACHE_PLANES=200000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_wc1big.csv $P > gpurun_out/${T}_ncu_wc1big.log 2>&1
python - <<'PY'
import csv, collections, os, re
T=os.environ.get("TAG","s4b")
for tag in ("wc0","wc1","wc1big"):
    f=f"gpurun_out/{T}_launches_{tag}.csv"
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
    print(tag)
    for k,(n,ms) in sorted(agg.items(), key=lambda x:-x[1][1])[:12]:
        print(f"   {ms:10.3f} ms {n:6d}  {k}")
PY
