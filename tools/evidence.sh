#!/bin/bash
# One GPU call that regenerates the round's evidence under gpurun_out/ev/:
# GPU tests, smoke, bench lines (default = C3, then C1 C2 C4 C5) + the
# reference arm, the launch list of the default bench command, ncu --set full
# captures (C3 64-view launch, C2 / C1 camera kernel, C4 hierarchy kernel, a
# C5 wave iteration) and the C5 per-launch DRAM traffic of one full step,
# cold (ncu's default cache flush per kernel) and warm (--cache-control none).
out=gpurun_out/ev; mkdir -p $out
python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; tail -1 $out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
python bench.py > $out/bench_default.json 2> $out/bench_default.err; tail -c 300 $out/bench_default.json
for c in c1 c2 c4 c5; do
  python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; tail -c 300 $out/bench_$c.json
done
python bench.py --impl reference > $out/bench_ref_default.json 2> $out/bench_ref_default.err; tail -c 200 $out/bench_ref_default.json
python bench.py --impl reference --config c2 > $out/bench_ref_c2.json 2> $out/bench_ref_c2.err; tail -c 200 $out/bench_ref_c2.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_default.csv python bench.py --steps 2 --warmup 3 > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:render_cameras_kernel -s 3 -c 1 -o $out/c3 -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:render_cameras_kernel -s 2 -c 1 -o $out/c2 -f python tools/run_once.py c2 nested > $out/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:render_cameras_kernel -s 3 -c 1 -o $out/c1 -f python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_c1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:render_hierarchy_kernel -s 3 -c 1 -o $out/c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 3 -c 1 -o $out/c5_wave -f python tools/c5_steps.py 24 1 > $out/ncu_c5.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $out/c5_traffic.csv python tools/c5_once.py > $out/ncu_c5t.log 2>&1
python tools/ncu_traffic_sum.py $out/c5_traffic.csv > $out/c5_traffic.txt
ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $out/c5_traffic_warm.csv python tools/c5_once.py > $out/ncu_c5tw.log 2>&1
python tools/ncu_traffic_sum.py $out/c5_traffic_warm.csv > $out/c5_traffic_warm.txt
rm -f $out/c5_traffic.csv $out/c5_traffic_warm.csv
# summaries on the box (the reports together exceed gpurun's 64 MiB return)
mkdir -p $out/summ
for c in c1 c2 c3 c4 c5_wave; do
  python tools/summarize_ncu.py $out/$c.ncu-rep $out/summ/r02_$c > $out/summ/${c}_dram_bytes.txt 2>&1
done
for c in c3 c5_wave c4 c2; do
  ncu -i $out/$c.ncu-rep --page source --csv --print-source=cuda,sass > $out/${c}_src.csv 2>/dev/null
  python tools/ncu_regions.py $out/${c}_src.csv > $out/summ/r02_${c}_functions.txt
  python tools/ncu_opcodes.py $out/${c}_src.csv > $out/summ/r02_${c}_opcodes.txt
  rm -f $out/${c}_src.csv
done
rm -f $out/c1.ncu-rep $out/c2.ncu-rep $out/c4.ncu-rep
ls -la $out $out/summ
