out=gpurun_out/r03t; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2" paper_2507_14624_b200/liblfprobe_b200.so $V/liblfprobe_b200_LFP_PIN_CF0.so $V/liblfprobe_b200_LFP_CHORD_SMEM_MAXB0.so $V/liblfprobe_b200_LFP_WALK_SMEM_MAXB0.so $V/liblfprobe_b200_LFP_CTA_WARPS2.so $V/liblfprobe_b200_LFP_CTA_WARPS8.so 2>&1 | tee $out/ab_retest2.txt
bash tools/ab.sh "c4" paper_2507_14624_b200/liblfprobe_b200.so $V/liblfprobe_b200_LFP_PIN_CF0.so $V/liblfprobe_b200_LFP_WALK_SMEM_HIER0.so $V/liblfprobe_b200_LFP_CHORD_SMEM_HIER0.so 2>&1 | tee -a $out/ab_retest2.txt
