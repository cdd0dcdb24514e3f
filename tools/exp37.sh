# class grids: PDL chain vs S side streams (and grid size)
mkdir -p gpurun_out
{
python tools/kbench.py 6:4:35:perm
for S in 2 4 8; do for d in 1 2 4; do HYGT_CLS_STREAMS=$S HYGT_CLS_GRID_DIV=$d python tools/kbench.py 6:4:35:perm; done; done
} > gpurun_out/exp37.log 2>&1
cat gpurun_out/exp37.log
