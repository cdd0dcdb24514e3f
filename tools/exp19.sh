# cls kernel: grid divisor sweep with next-batch prefetch
mkdir -p gpurun_out
{
for d in 1 2 3 4 6; do HYGT_CLS_GRID_DIV=$d python tools/kbench.py 6:4:35:perm; done
} > gpurun_out/exp19.log 2>&1
cat gpurun_out/exp19.log
