# round-1 profile pass of the default bench command (launch list incl. configs 3 and 5)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_default.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_default.log 2>&1
echo rc=$?
ls -la gpurun_out/launches_default.csv
