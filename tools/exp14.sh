K="timeout 300 python tools/kbench.py"
for L in __ldg __ldcs; do HYGT_JIT_LOAD=$L $K 4:3:35:perm 4:3:1:perm; done
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "golden_float or config_shapes or edge" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
