mkdir -p gpurun_out
for c in 2 3; do
python bench.py --config $c --profile-steps 2 > gpurun_out/plain$c.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_predict --csv --log-file gpurun_out/pred_$c.csv python bench.py --config $c --profile-steps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:k_predict --csv --log-file gpurun_out/predw_$c.csv python bench.py --config $c --profile-steps 2 > /dev/null 2>&1
done
for f in gpurun_out/pred_*.csv gpurun_out/predw_*.csv; do echo $f; grep k_predict $f | awk -F'","' '{print $13, $15}'; done
