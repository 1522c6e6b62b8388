out=gpurun_out/r02i; mkdir -p $out
V=build/variants
bash tools/ab.sh "c5 c3 c2" $V/liblfprobe_b200_LFP_SEG_WW0.so $V/liblfprobe_b200_LFP_HI_PREFETCH1.so $V/liblfprobe_b200_LFP_HI_PREFETCH1_LFP_TILED1.so $V/liblfprobe_b200_LFP_HI_PREFETCH0_LFP_TILED1.so $V/liblfprobe_b200_LFP_HI_PREFETCH1_LFP_SEG_WW3.so 2>&1 | tee $out/ab_pf.txt
