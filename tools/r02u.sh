out=gpurun_out/r02u; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c5" $V/liblfprobe_b200_LFP_FAST_DIV1.so $V/liblfprobe_b200_LFP_FAST_DIV2.so $V/liblfprobe_b200_LFP_FAST_DIV3.so 2>&1 | tee $out/ab_fastdiv.txt
ncu --set full --clock-control none --import-source on -k regex:render_cameras_kernel -s 3 -c 1 -o $out/c3 -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 3 -c 1 -o $out/c5_wave -f python tools/c5_steps.py 24 1 > $out/ncu_c5.log 2>&1
