# clsjit N = 64 / 32: minimum resident CTAs (register cap) sweep
mkdir -p gpurun_out
for m in 12 16 20 24; do HYGT_CLS_MINB=$m python tools/kbench.py 6:4:35:perm 5:3:35:perm; done > gpurun_out/exp33.log 2>&1
cat gpurun_out/exp33.log
