# round 3a: cluster-split narrow levels (existing cluster code, more warps per CTA)
# A/B on configs 1 and 2 (fp64 device ms), plus parity of the cluster variant
mkdir -p gpurun_out
out=gpurun_out/r3a_ab.txt
: > $out
for c in 1 2; do
  for v in "main:" "cl6:2" "cl6:4" "clw:2" "clw:4"; do
    tag=${v%%:*}; cl=${v#*:}
    lib=""; [ "$tag" != main ] && lib=paper_2207_00233_b200/variants/libfse_b200_$tag.so
    FSE_LIB=$lib FSE_CLUSTER=$cl timeout 300 python bench.py --config $c --steps 10 --warmup 3 > /tmp/r3a.json 2>/tmp/r3a.err
    python -c "
import json;d=json.loads(open('/tmp/r3a.json').read().strip().splitlines()[-1])
print('config $c', '$tag', 'CL=$cl', {k: round(v['ms'],3) for k,v in d['runs'].items()})" >> $out 2>&1 || tail -3 /tmp/r3a.err >> $out
  done
done
FSE_LIB=paper_2207_00233_b200/variants/libfse_b200_clw.so FSE_CLUSTER=2 timeout 600 python -m pytest tests/test_gpu_conceal.py -m gpu -x -q -k "golden or full" > gpurun_out/r3a_pytest_clw2.log 2>&1
echo "pytest clw CL=2 rc=$?" >> $out; tail -2 gpurun_out/r3a_pytest_clw2.log >> $out
cat $out
