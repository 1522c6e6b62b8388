out=gpurun_out/r02k; mkdir -p $out
V=build/variants
for rep in 1 2; do for lib in $V/liblfprobe_b200_LFP_WAVE_KEY_LEN0.so $V/liblfprobe_b200_LFP_WAVE_KEY_LEN1.so; do
  LFP_LIB_PATH=$lib timeout 300 python tools/c5_steps.py 26 3 2>&1 | tail -1 | tee -a $out/ab_len.txt
done; done
which compute-sanitizer; compute-sanitizer --version 2>&1 | head -3
timeout 900 bash tools/sanitize.sh $out/sanitize; echo sanitize rc=$?
