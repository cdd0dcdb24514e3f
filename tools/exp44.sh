mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k correlation 2>&1 | tail -2
for c in 2 3 5; do timeout 300 python tools/corr_bench.py --config $c; done
