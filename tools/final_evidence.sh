mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r02z_bench.log 2>&1
nvidia-smi -q -d CLOCK,PERFORMANCE > gpurun_out/r02z_smi.txt 2>&1
python tools/mass_drift.py > gpurun_out/r02z_drift.log 2>&1
python tools/bench_scenes.py > gpurun_out/r02z_scenes.jsonl 2> gpurun_out/r02z_scenes.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02z_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r02z_ncu_launch.log 2>&1
python tools/prof_step.py 512 q16 4 > gpurun_out/r02z_prof_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fluid_interior -s 2 -c 1 -o gpurun_out/r02z_q16 python tools/prof_step.py 512 q16 4 > gpurun_out/r02z_ncu_q16.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fluid_interior -s 2 -c 1 -o gpurun_out/r02z_fp32 python tools/prof_step.py 512 fp32 4 > gpurun_out/r02z_ncu_fp32.log 2>&1
echo done > gpurun_out/r02z_done
