out=gpurun_out/r02g; mkdir -p $out
V=build/variants
for v in 0 3; do
LFP_LIB_PATH=$V/liblfprobe_b200_LFP_SEG_WW$v.so ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 3 -c 1 -o $out/c5_ww$v -f python tools/c5_steps.py 24 1 > $out/ncu_c5_ww$v.log 2>&1
done
ls -la $out
