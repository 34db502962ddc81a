# (--cache-control none on the window-launch captures: a sweep is ~600 chained launches that find
# the operands in L2; flushing the caches before the profiled launch would count a cold refill of
# the whole working set as that launch's DRAM traffic)
# Round-1 measurement capture (run under gpurun): bench line, launch list of the same command,
# ncu --set full of the two main sweep kernels, pytest -m gpu. Summaries: tools/ncu_summary.py.
#   bash tools/capture_r01.sh <tag>      (tag e.g. r01_v14)
TAG=${1:-r01_v14}
set -x
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_l.log 2>&1
python tools/time_c4.py C4aamp > /dev/null && ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled -k 'regex:sweep_kernel_rc<mpg::Wide<mpg::EuclidCov' -s 40 -c 1 -o gpurun_out/aamp python tools/time_c4.py C4aamp > gpurun_out/ncu_a.log 2>&1
python tools/time_c4.py C4acamp > /dev/null && ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled -k 'regex:sweep_kernel_rc<mpg::Wide<mpg::Znorm<\(bool\)0>' -s 40 -c 1 -o gpurun_out/acamp python tools/time_c4.py C4acamp > gpurun_out/ncu_z.log 2>&1
python tools/time_c4.py C4aamp C4acamp C5 C2 C3p1 C3p3 C1 > gpurun_out/time_c4.json 2>&1
# summarise on the box (two --set full reports exceed gpurun's 64 MiB copy-back limit)
python tools/ncu_summary.py $TAG --launches gpurun_out/launches.csv --rep gpurun_out/aamp.ncu-rep --rep gpurun_out/acamp.ncu-rep > gpurun_out/summary.log 2>&1
# DRAM traffic of the window launches from a single-pass run (tools/window_traffic.py says why)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/win_traffic.csv --kernel-name-base demangled -k regex:sweep_kernel_rc -s 60 -c 300 python tools/time_c4.py C4aamp C4acamp > gpurun_out/win_traffic.log 2>&1
python tools/window_traffic.py gpurun_out/win_traffic.csv $TAG >> gpurun_out/summary.log 2>&1
cp profiles/${TAG}_* profiles/ncu_summary.json gpurun_out/
rm -f gpurun_out/acamp.ncu-rep
ls -la gpurun_out
