K="timeout 200 python tools/kbench.py"
export HYGT_TILE_L=1 HYGT_TILE_VPT=2 HYGT_TILE_ROWS=4096
for P in 0 1 2 3; do export HYGT_LOAD_POLICY=$P; echo "policy $P"; $K 4:1:35:noperm:rand 4:3:35:perm:rand; done
