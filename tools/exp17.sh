K="timeout 300 python tools/kbench.py"
for LV in "1 2" "2 12" "1 10"; do set -- $LV; HYGT_TILE_L=$1 HYGT_TILE_VPT=$2 $K 4:3:35:perm; done
