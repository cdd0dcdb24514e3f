K="timeout 200 python tools/kbench.py"
export HYGT_TILE_L=1 HYGT_TILE_VPT=2 HYGT_TILE_ROWS=4096
$K 4:1:35:noperm:rand 4:1:35:noperm:sorted 4:1:35:noperm:zero 4:1:35:noperm:runs64 4:1:2:noperm:rand 4:1:1:noperm:zero
