# A/B of narrow-level variant builds (variants/libfse_b200_<tag>.so built with -DFSE_CLOCKS):
# lone-window clock breakdown, fp32 and fp64 (12-warp fp64 narrow variant)
mkdir -p gpurun_out
for t in ${TAGS:-base lg3 lg6 lg6m1 lg3m1}; do
  FSE_LIB=paper_2207_00233_b200/variants/libfse_b200_$t.so FSE_F64L=12 python tools/clock_breakdown.py fp32 fp64 \
    | sed "s/^{/{\"tag\": \"$t\", /" >> gpurun_out/${OUT:-narrow_ab}.jsonl 2>&1
done
