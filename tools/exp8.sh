K="timeout 200 python tools/kbench.py"
for LV in "1 2" "2 2" "0 1"; do set -- $LV; export HYGT_TILE_L=$1 HYGT_TILE_VPT=$2
for T in 4096 8192; do export HYGT_TILE_ROWS=$T; $K 4:1:35:noperm:rand 4:3:35:perm:rand 4:3:35:perm:sorted; done; done
