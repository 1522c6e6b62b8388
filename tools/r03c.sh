out=gpurun_out/r03c; mkdir -p $out
V=build/variants
bash tools/ab.sh "c5 c3" $V/liblfprobe_b200_LFP_SEG_WW0.so $V/liblfprobe_b200_LFP_SEG_WW1.so $V/liblfprobe_b200_LFP_SEG_WW2.so $V/liblfprobe_b200_LFP_SEG_WW3.so 2>&1 | tee $out/ab_ww2.txt
