# stage kernel: L2 evict_first cache policy on the row copies (bit0 loads, bit1 stores)
mkdir -p gpurun_out
for i in 1 2; do for h in 0 1 2 3; do HYGT_STAGE_L2HINT=$h timeout 300 python bench.py --steps 20 --no-e2e --no-cpu --no-extra | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('l2hint=$h', d['value'], round(d['roofline']['frac'],4), d['breakdown_ms'])"; done; done
