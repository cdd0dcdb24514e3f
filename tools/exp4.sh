mkdir -p gpurun_out
K="timeout 200 python tools/kbench.py"
{
for LV in "1 2" "2 2" "0 1"; do set -- $LV; export HYGT_TILE_L=$1 HYGT_TILE_VPT=$2 HYGT_TILE_ROWS=4096
  $K 4:3:1:noperm 4:3:1:perm 4:3:35:noperm 4:3:35:perm 4:1:1:noperm 4:1:35:noperm
done
export HYGT_TILE=0; unset HYGT_TILE_L HYGT_TILE_VPT HYGT_TILE_ROWS
$K 4:3:1:noperm 4:1:1:noperm
} > gpurun_out/exp4.log 2>&1
cat gpurun_out/exp4.log
