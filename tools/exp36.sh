mkdir -p gpurun_out
for d in 1 2 3 4; do HYGT_CLS_GRID_DIV=$d python tools/kbench.py 6:4:35:perm 5:3:35:perm; done > gpurun_out/exp36.log 2>&1
cat gpurun_out/exp36.log
