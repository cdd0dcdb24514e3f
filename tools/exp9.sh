K="timeout 200 python tools/kbench.py"
for LV in "1 2" "2 2" "2 4"; do set -- $LV; export HYGT_TILE_L=$1 HYGT_TILE_VPT=$2 HYGT_TILE_ROWS=4096
$K 4:3:35:perm:rand 4:3:1:noperm:zero; done
