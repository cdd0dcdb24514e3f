K="timeout 300 python tools/kbench.py"
for CH in 262144 0 65536; do HYGT_CHUNK_ROWS=$CH $K 4:3:35:perm:rand; done
$K 4:3:1:perm 4:3:8:perm
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench.log 2>&1; head -c 1100 gpurun_out/bench.log; echo
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
