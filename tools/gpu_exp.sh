mkdir -p gpurun_out
PAC_SRT_HASH_KERNEL=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_sort_nohash.csv python tools/prof_agg.py --config C3 --iters 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_srt_scatter" -c 2 -o gpurun_out/srt_p0 -f python tools/prof_agg.py --config C3 --iters 1 > gpurun_out/ncu_p0.log 2>&1; echo "ncu rc=$?"
