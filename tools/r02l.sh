out=gpurun_out/r02l; mkdir -p $out
V=build/variants
for rep in 1 2; do for lib in $V/liblfprobe_b200_LFP_WAVE_PACKED0.so $V/liblfprobe_b200_LFP_WAVE_PACKED1.so $V/liblfprobe_b200_LFP_WAVE_PACKED1_LFP_WAVE_RELOAD_RAY1.so; do
  LFP_LIB_PATH=$lib timeout 300 python tools/c5_steps.py 26 3 2>&1 | tail -1 | tee -a $out/ab_packed.txt
done; done
python -m pytest tests -m gpu -q -x -k "wave or C5 or c5 or bounds or sharded" > $out/pytest_wave.log 2>&1; tail -3 $out/pytest_wave.log
for v in 0 1; do
LFP_LIB_PATH=$V/liblfprobe_b200_LFP_WAVE_PACKED$v.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $out/c5_traffic_packed$v.csv python tools/c5_once.py > $out/ncu_c5t_$v.log 2>&1
python tools/ncu_traffic_sum.py $out/c5_traffic_packed$v.csv | tee $out/c5_traffic_packed$v.txt
done
LFP_LIB_PATH=$V/liblfprobe_b200_LFP_WAVE_PACKED1.so ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $out/c5_traffic_packed1_warm.csv python tools/c5_once.py > $out/ncu_c5t_1w.log 2>&1
python tools/ncu_traffic_sum.py $out/c5_traffic_packed1_warm.csv | tee $out/c5_traffic_packed1_warm.txt
