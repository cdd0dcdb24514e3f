set -x
mkdir -p gpurun_out/c1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "correlation" > gpurun_out/c1/test.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/c1/test.log
for c in 3 5; do timeout 300 python tools/corr_bench.py --config $c --steps 5 > gpurun_out/c1/corr_cfg$c.json 2>&1; echo "bench $c rc=$?"; cat gpurun_out/c1/corr_cfg$c.json | head -c 600; echo; done
timeout 300 python tools/corr_bench.py --config 5 --steps 2 --knob HYGT_CORR_TC=0 > gpurun_out/c1/corr_cfg5_simt.json 2>&1; head -c 400 gpurun_out/c1/corr_cfg5_simt.json
