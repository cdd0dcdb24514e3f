# next-batch prefetch mode: 0 none, 1 bulk (UBLKPF uniform loop), 2 per-lane prefetch.global.L2
mkdir -p gpurun_out
{
for m in 1 0 2; do HYGT_FIXED_PF=$m python tools/fixed_bench.py --config 2 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fixed cfg2 pf=$m', d['value'], d['ms_fwd'])"; done
for m in 1 0 2; do HYGT_FIXED_PF=$m python tools/fixed_bench.py --config 3 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fixed cfg3 pf=$m', d['value'], d['ms_fwd'])"; done
for m in 1 0 2; do HYGT_CLS_PF=$m python tools/kbench.py 5:3:35:perm 6:4:35:perm; done
} > gpurun_out/exp35.log 2>&1
cat gpurun_out/exp35.log
