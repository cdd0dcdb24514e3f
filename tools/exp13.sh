K="timeout 300 python tools/kbench.py"
for L in __ldcs __ldg ld_l2_128 ld_l2_256; do HYGT_JIT_LOAD=$L $K 4:3:35:perm; done
timeout 300 python tools/kbench.py 4:3:35:perm > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:hygt_jit -s 3 -c 1 -o /tmp/pj python tools/kbench.py 4:3:35:perm > gpurun_out/ncu_j.log 2>&1
ncu -i /tmp/pj.ncu-rep --page raw --csv > gpurun_out/prof_jit_raw.csv 2>/dev/null
