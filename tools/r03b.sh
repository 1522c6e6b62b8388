out=gpurun_out/r03b; mkdir -p $out
V=build/variants
bash tools/ab.sh "c5" $V/liblfprobe_b200_LFP_WAVE_CELL_BITS6.so $V/liblfprobe_b200_LFP_WAVE_CELL_BITS5.so $V/liblfprobe_b200_LFP_WAVE_CELL_BITS4.so $V/liblfprobe_b200_LFP_ALIGN_FILTER1.so 2>&1 | tee $out/ab_bits.txt
bash tools/ab.sh "c3" $V/liblfprobe_b200_LFP_WAVE_CELL_BITS6.so $V/liblfprobe_b200_LFP_ALIGN_FILTER1.so 2>&1 | tee -a $out/ab_bits.txt
