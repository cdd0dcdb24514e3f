# clsjit N = 64: double-buffered slots vs single
mkdir -p gpurun_out
{
python tools/kbench.py 6:4:35:perm
HYGT_CLS_DB=1 python tools/kbench.py 6:4:35:perm
python tools/kbench.py 5:3:35:perm
HYGT_CLS_DB=1 python tools/kbench.py 5:3:35:perm
} > gpurun_out/exp29.log 2>&1
HYGT_CLS_DB=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "seg2_path or config_shapes" 2>&1 | tail -2
cat gpurun_out/exp29.log
