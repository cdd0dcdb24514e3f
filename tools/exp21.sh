# per-class NVRTC kernels (clsjit) vs parameter-table kernels (cls) vs seg2, cfg3 shape
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "seg2_path or golden_float or config_shapes or coexist" > gpurun_out/pt21.log 2>&1; echo rc=$? >> gpurun_out/pt21.log
{
python tools/kbench.py 6:4:35:perm
HYGT_CLS_JIT=0 python tools/kbench.py 6:4:35:perm
} > gpurun_out/exp21.log 2>&1
timeout 300 python bench.py --config 3 --steps 10 --no-e2e --no-cpu > gpurun_out/b3_jit.json 2>gpurun_out/b3_jit.err
tail -3 gpurun_out/pt21.log; cat gpurun_out/exp21.log gpurun_out/b3_jit.json
