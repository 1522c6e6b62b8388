out=gpurun_out/r02j; mkdir -p $out
V=build/variants
for rep in 1 2; do for lib in $V/liblfprobe_b200_LFP_SEG_WW0.so $V/liblfprobe_b200_LFP_WAVE_CTA32.so $V/liblfprobe_b200_LFP_WAVE_CTA64.so $V/liblfprobe_b200_LFP_WAVE_CTA256.so; do
  LFP_LIB_PATH=$lib timeout 300 python tools/c5_steps.py 26 3 2>&1 | tail -1 | tee -a $out/ab_cta.txt
done; done
