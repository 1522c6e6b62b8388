out=gpurun_out/r02h; mkdir -p $out
V=build/variants
bash tools/ab.sh "c5 c3 c2" $V/liblfprobe_b200_LFP_SEG_WW0.so $V/liblfprobe_b200_LFP_SEG_WW1.so $V/liblfprobe_b200_LFP_SEG_WW2.so $V/liblfprobe_b200_LFP_SEG_WW3.so 2>&1 | tee $out/ab_ww.txt
LFP_LIB_PATH=$V/liblfprobe_b200_LFP_SEG_WW3.so ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 3 -c 1 -o $out/c5_ww3 -f python tools/c5_steps.py 24 1 > $out/ncu_c5_ww3.log 2>&1
