# KLT: raw cp.async row staging (two tiles in flight) vs register prefetch
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k klt 2>&1 | tail -2
for i in 1 2; do for r in 1 0; do HYGT_KLT_RAW=$r timeout 300 python bench.py --config 4 --steps 10 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('raw=$r', d['roofline']['frac'], d['ms_per_step'], d['roundtrip_max_rel'])"; done; done
