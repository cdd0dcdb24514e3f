mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden_float or config_shapes or energy" > gpurun_out/pt256b.log 2>&1; echo rc=$? >> gpurun_out/pt256b.log
tail -3 gpurun_out/pt256b.log
HYGT_CLS_JIT256=1 timeout 400 python bench.py --config 5 --steps 10 --no-e2e --no-cpu > gpurun_out/b5_jit.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b5_jit.json').read().strip().splitlines()[-1]); print(d['config']['kernel_path'], d['roofline']['frac'], d['breakdown_ms'])"
