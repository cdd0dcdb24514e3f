mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k correlation 2>&1 | tail -2
for e in 8 4; do for c in 3 5; do HYGT_CORR_E=$e timeout 300 python tools/corr_bench.py --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('E=$e', d['workload'], d['value'], d['ms'])"; done; done
