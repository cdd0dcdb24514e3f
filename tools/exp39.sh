# e2e (HostPipeline) chunk size / stream count sweep on config 2
mkdir -p gpurun_out
for ch in 1048576 2097152 4194304; do for s in 2 4 6; do
HYGT_E2E_CHUNK=$ch HYGT_E2E_STREAMS=$s timeout 300 python bench.py --steps 5 --no-cpu --no-extra | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk=$ch streams=$s', round(d['e2e']['value']/1e6,1), 'M vec/s', round(d['e2e']['ms_per_step'],2), 'ms')"
done; done > gpurun_out/exp39.log 2>&1
cat gpurun_out/exp39.log
