# cls kernel: chain vs single big launch, and a full ncu capture of one big class launch
mkdir -p gpurun_out
{
python tools/kbench.py 6:4:35:perm 6:4:35:perm:zero 6:4:35:perm:sorted 6:4:4:perm
HYGT_CLS=0 python tools/kbench.py 6:4:35:perm 6:4:35:perm:zero
} > gpurun_out/exp18.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hygt_cls_kernel -s 105 -c 1 -f -o /tmp/cls_zero python tools/kbench.py 6:4:35:perm:zero > gpurun_out/ncu_cls.log 2>&1
ncu -i /tmp/cls_zero.ncu-rep --page raw --csv > gpurun_out/cls_zero_raw.csv 2>/dev/null
ncu -i /tmp/cls_zero.ncu-rep --page details --csv > gpurun_out/cls_zero_details.csv 2>/dev/null
ncu -i /tmp/cls_zero.ncu-rep --page source --csv --print-source sass > gpurun_out/cls_zero_source.csv 2>/dev/null
cat gpurun_out/exp18.log
