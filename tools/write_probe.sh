python tools/write_probe.py > gpurun_out/write_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/write_probe_ncu.csv python tools/write_probe.py > /dev/null 2>&1
