out=gpurun_out/r02y; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2 c5" $V/liblfprobe_b200_LFP_FLOOR_CVT0.so $V/liblfprobe_b200_LFP_FLOOR_CVT1.so 2>&1 | tee $out/ab_floor.txt
bash tools/ab.sh "c5" $V/liblfprobe_b200_LFP_WAVE_CF_SMEM0.so 2>&1 | tee -a $out/ab_floor.txt
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
python bench.py --config c5 --steps 3 --warmup 3 > $out/bench_c5.json 2>$out/bench_c5.err; tail -c 700 $out/bench_c5.json
