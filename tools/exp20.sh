# cls kernel: rows per thread (VPT) and grid divisor
mkdir -p gpurun_out
{
for v in 1 2; do for d in 1 2; do HYGT_CLS_VPT=$v HYGT_CLS_GRID_DIV=$d python tools/kbench.py 6:4:35:perm; done; done
HYGT_CLS_VPT=2 python tools/kbench.py 6:4:35:perm:zero
} > gpurun_out/exp20.log 2>&1
cat gpurun_out/exp20.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "seg2_path or config_shapes" 2>&1 | tail -3
