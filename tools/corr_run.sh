# correlation kernels on the GPU box: parity tests, timings at config 3 (N=64) and 5 (N=256)
out=${1:-gpurun_out/c}
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "correlation" > $out/test.log 2>&1; echo "pytest rc=$?"; tail -3 $out/test.log
for c in 3 5; do timeout 300 python tools/corr_bench.py --config $c --steps 5 > $out/corr_cfg$c.json 2>&1; echo "bench $c rc=$?"; head -c 300 $out/corr_cfg$c.json; echo; done
