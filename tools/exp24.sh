# instruction-cache probe: per-class NVRTC kernels with 4x / 2x the code of config 3 (R = 16, 8)
mkdir -p gpurun_out
{
python tools/kbench.py 6:4:4:perm 6:8:4:perm 6:16:4:perm
} > gpurun_out/exp24.log 2>&1
cat gpurun_out/exp24.log
