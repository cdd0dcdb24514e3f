# One full ncu capture of one kernel launch of an arbitrary command (exported to CSV on the box).
#   bash tools/prof_cmd.sh NAME KERNEL_REGEX LAUNCH_SKIP COMMAND...
name=$1; regex=$2; skip=$3; shift 3
mkdir -p gpurun_out
timeout 300 "$@" > gpurun_out/plain_$name.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$regex" -s $skip -c 1 -f -o /tmp/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof_${name}_raw.csv 2>/dev/null
ncu -i /tmp/prof_$name.ncu-rep --page details --csv > gpurun_out/prof_${name}_details.csv 2>/dev/null
ncu -i /tmp/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${name}_sass.csv 2>/dev/null
