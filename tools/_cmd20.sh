python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02_c3_plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_c3_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu1.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc2_kernel -c 5 --csv --log-file gpurun_out/r02_c3_traffic.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc2_kernel -c 5 -o gpurun_out/r02_c3_tc2_full python bench.py --rows 1000000 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu3.log 2>&1
echo done
