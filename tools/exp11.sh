K="timeout 300 python tools/kbench.py"
$K 4:3:35:perm 4:3:1:noperm:zero 4:3:1:perm
HYGT_JIT=0 $K 4:3:35:perm
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
