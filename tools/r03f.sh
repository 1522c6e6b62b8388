out=gpurun_out/r03f; mkdir -p $out
V=build/variants
bash tools/ab.sh "c5" paper_2507_14624_b200/liblfprobe_b200.so $V/liblfprobe_b200_LFP_HI_PREFETCH1.so $V/liblfprobe_b200_LFP_WAVE_MIN_BLOCKS8.so $V/liblfprobe_b200_LFP_WAVE_CF_SMEM0.so $V/liblfprobe_b200_LFP_TILED1.so $V/liblfprobe_b200_LFP_WAVE_CTA32.so $V/liblfprobe_b200_LFP_WAVE_CTA128.so $V/liblfprobe_b200_LFP_WAVE_CHORD_SMEM0.so 2>&1 | tee $out/ab_retest.txt
bash tools/ab.sh "c3" paper_2507_14624_b200/liblfprobe_b200.so $V/liblfprobe_b200_LFP_HI_PREFETCH1.so $V/liblfprobe_b200_LFP_TILED1.so 2>&1 | tee -a $out/ab_retest.txt
