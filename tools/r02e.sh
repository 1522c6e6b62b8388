out=gpurun_out/r02e; mkdir -p $out
V=build/variants
for rep in 1 2; do for lib in $V/liblfprobe_b200_LFP_WAVE_KEY_NSEG0.so $V/liblfprobe_b200_LFP_WAVE_KEY_NSEG1.so; do
  LFP_LIB_PATH=$lib timeout 300 python tools/c5_steps.py 26 3 2>&1 | tail -1 | tee -a $out/ab_nseg.txt
done; done
