export HYGT_TILE_L=1 HYGT_TILE_VPT=2 HYGT_TILE_ROWS=4096
timeout 200 python tools/kbench.py 4:1:35:noperm:rand 4:1:35:noperm:sorted > gpurun_out/k7.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:hygt_tile_kernel -s 3 -c 1 -o gpurun_out/prof_rand python tools/kbench.py 4:1:35:noperm:rand > gpurun_out/ncu7a.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:hygt_tile_kernel -s 3 -c 1 -o gpurun_out/prof_sorted python tools/kbench.py 4:1:35:noperm:sorted > gpurun_out/ncu7b.log 2>&1
cat gpurun_out/k7.log
