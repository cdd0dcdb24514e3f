# clsjit / cls: per-lane L2 prefetch of the next batch vs none
mkdir -p gpurun_out
{
python tools/kbench.py 6:4:35:perm
HYGT_CLS_PREFETCH=0 python tools/kbench.py 6:4:35:perm
HYGT_CLS_JIT=0 python tools/kbench.py 6:4:35:perm
} > gpurun_out/exp23.log 2>&1
cat gpurun_out/exp23.log
