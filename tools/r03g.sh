out=gpurun_out/r03g; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2" paper_2507_14624_b200/liblfprobe_b200.so $V/liblfprobe_b200_LFP_CFS_MINB4.so $V/liblfprobe_b200_LFP_CFS_MINB4_LFP_MIN_BLOCKS5.so 2>&1 | tee $out/ab_cfs.txt
