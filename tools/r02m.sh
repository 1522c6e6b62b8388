out=gpurun_out/r02m; mkdir -p $out
V=build/variants
for rep in 1 2; do for lib in $V/liblfprobe_b200_LFP_WAVE_MIN_BLOCKS7.so $V/liblfprobe_b200_LFP_WAVE_MIN_BLOCKS6.so $V/liblfprobe_b200_LFP_WAVE_MIN_BLOCKS8.so $V/liblfprobe_b200_LFP_WAVE_MIN_BLOCKS7_LFP_WAVE_CHORD_SMEM0.so $V/liblfprobe_b200_LFP_WAVE_MIN_BLOCKS8_LFP_WAVE_CHORD_SMEM0.so $V/liblfprobe_b200_LFP_WAVE_MIN_BLOCKS7_LFP_WAVE_CTA32.so; do
  LFP_LIB_PATH=$lib timeout 300 python tools/c5_steps.py 26 3 2>&1 | tail -1 | tee -a $out/ab_occ.txt
done; done
