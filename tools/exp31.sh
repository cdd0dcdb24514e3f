# stage sort: CTA per tile vs warp per tile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stage or golden_float or config_shapes or bucketing or fixed or invalid" > gpurun_out/pt_sort2.log 2>&1; echo rc=$? >> gpurun_out/pt_sort2.log
tail -3 gpurun_out/pt_sort2.log
for i in 1 2; do
for v in 1 0; do HYGT_SORT2=$v timeout 300 python bench.py --steps 20 --no-e2e --no-cpu --no-extra | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sort2=$v', d['value'], d['breakdown_ms'])"; done
done
