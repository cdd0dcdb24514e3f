# One full ncu capture of one kernel launch, exported to CSV on the box.
#   bash tools/prof_one.sh NAME KERNEL_REGEX "BENCH ARGS"
mkdir -p gpurun_out
timeout 300 python bench.py $3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_$1.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 4 -c 1 -f -o /tmp/prof_$1 \
  python bench.py $3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$1.log 2>&1
ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1_raw.csv 2>/dev/null
ncu -i /tmp/prof_$1.ncu-rep --page details --csv > gpurun_out/prof_$1_details.csv 2>/dev/null
ncu -i /tmp/prof_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$1_sass.csv 2>/dev/null
ls -la gpurun_out/prof_$1_*
