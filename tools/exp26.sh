# fixed point: per-class NVRTC chain vs staged / row kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_apply.py -m gpu -x -q -k "fixed or apply" > gpurun_out/pt_fx.log 2>&1; echo rc=$? >> gpurun_out/pt_fx.log
{
timeout 300 python tools/fixed_bench.py --config 2
HYGT_FIXED_JIT=0 timeout 300 python tools/fixed_bench.py --config 2
timeout 300 python tools/fixed_bench.py --config 3
HYGT_FIXED_JIT=0 timeout 300 python tools/fixed_bench.py --config 3
} > gpurun_out/exp26.log 2>&1
tail -4 gpurun_out/pt_fx.log; cat gpurun_out/exp26.log
