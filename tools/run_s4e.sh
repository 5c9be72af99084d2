# clock64 phase breakdown (3 windows per SM): previous tree, this tree computing W, this tree with cached W
mkdir -p gpurun_out
T=${TAG:-s4e}
ROOT=$PWD
(cd ab_base && WINDOWS=444 FSE_LIB=$PWD/paper_2207_00233_b200/variants/libfse_b200_clk.so python tools/clock_breakdown.py fp64 > $ROOT/gpurun_out/${T}_base.jsonl 2>&1)
WINDOWS=444 FSE_WCACHE=0 FSE_LIB=$PWD/paper_2207_00233_b200/variants/libfse_b200_clk.so python tools/clock_breakdown.py fp64 > gpurun_out/${T}_wc0.jsonl 2>&1
WINDOWS=444 FSE_WCACHE=1 FSE_WCACHE_ENTRIES=1 FSE_LIB=$PWD/paper_2207_00233_b200/variants/libfse_b200_clk.so python tools/clock_breakdown.py fp64 > gpurun_out/${T}_wc1.jsonl 2>&1
tail -2 gpurun_out/${T}_base.jsonl gpurun_out/${T}_wc0.jsonl gpurun_out/${T}_wc1.jsonl
