out=gpurun_out/r02c; mkdir -p $out
V=build/variants
for rep in 1 2; do
for lib in paper_2507_14624_b200/liblfprobe_b200.so $V/liblfprobe_b200_LFP_WAVE_STREAMING0_LFP_WAVE_L2_PERSIST0.so $V/liblfprobe_b200_LFP_WAVE_STREAMING1_LFP_WAVE_L2_PERSIST0.so $V/liblfprobe_b200_LFP_WAVE_STREAMING0_LFP_WAVE_L2_PERSIST1.so; do
  LFP_LIB_PATH=$lib timeout 300 python tools/c5_steps.py 26 3 2>&1 | tail -1 | tee -a $out/ab_wave.txt
done; done
ncu --set full --clock-control none --import-source on -k regex:render_cameras_kernel -s 3 -c 1 -o $out/c3 -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 3 -c 1 -o $out/c5_wave -f python tools/c5_steps.py 24 1 > $out/ncu_c5.log 2>&1
ls -la $out
