timeout 900 python -m pytest tests/test_gpu_aamp_cov.py tests/test_gpu_peer_merge.py -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
python tools/time_bands.py C4 1 2 4 8 > gpurun_out/bands_c4.log 2>&1
python tools/time_bands.py C5 1 2 4 8 > gpurun_out/bands_c5.log 2>&1
tail -1 gpurun_out/bands_c4.log | head -c 300
