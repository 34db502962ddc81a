set -x
python bench.py > gpurun_out/bench_r01_v11.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_l.log 2>&1
python tools/time_c4.py C4aamp > /dev/null && ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/aamp python tools/time_c4.py C4aamp > gpurun_out/ncu_a.log 2>&1
python tools/time_c4.py C4acamp > /dev/null && ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/acamp python tools/time_c4.py C4acamp > gpurun_out/ncu_z.log 2>&1
MPROF_PRECISION=fp32 python tools/time_cfg.py c4 1048576 1024 e; MPROF_PRECISION=fp32 python tools/time_cfg.py c4 1048576 1024 z
ls -la gpurun_out
