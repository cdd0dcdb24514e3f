K="timeout 300 python tools/kbench.py"
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for V in 0 1 2 3; do HYGT_SEG_VARIANT=$V $K 6:4:35:perm; done
for V in 6 7 8 9; do HYGT_SEG_VARIANT=$V $K 8:4:35:noperm; done
HYGT_SEGMENT=0 $K 6:4:35:perm 8:4:35:noperm
