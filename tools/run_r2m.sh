mkdir -p gpurun_out
export FSE_LIB=paper_2207_00233_b200/variants/libfse_b200_clk.so
B=8 F=128 python tools/clock_breakdown.py fp64 fp32 > gpurun_out/r2m_clk.jsonl 2>&1
B=8 F=128 WINDOWS=296 python tools/clock_breakdown.py fp64 fp32 >> gpurun_out/r2m_clk.jsonl 2>&1
FSE_TRACK_BELOW=0 python tools/clock_breakdown.py fp32 | sed 's/^{/{"lazy6": 1, /' >> gpurun_out/r2m_clk.jsonl 2>&1
