# per-class NVRTC chain for N = 16 (config 2 shape) vs the staged kernel
mkdir -p gpurun_out
{
python tools/kbench.py 4:3:35:perm
HYGT_CLS_JIT_SHORT=1 HYGT_STAGE=0 HYGT_TILE=0 python tools/kbench.py 4:3:35:perm
HYGT_CLS_JIT_SHORT=1 HYGT_STAGE=0 HYGT_TILE=0 python tools/kbench.py 5:3:35:perm
python tools/kbench.py 5:3:35:perm
} > gpurun_out/exp25.log 2>&1
cat gpurun_out/exp25.log
