for l in build/variants/old.so build/variants/libmprof_gpu_d8_t128_s128_b4.so build/variants/libmprof_gpu_d8_t128_s128_b4_ws_t256.so build/variants/libmprof_gpu_d8_t128_s128_b4_ws_t64.so; do
 for c in C4aamp C4acamp C5; do
  echo -n "$(basename $l) $c "; MPROF_GPU_LIB=$l ncu --metrics gpu__time_duration.sum --clock-control none -k regex:_stats --csv python tools/time_c4.py $c 2>/dev/null | grep -E "_stats" | awk -F, '{print $NF}' | tr -d '"' | sort -n | awk '{a[NR]=$1} END{print a[int((NR+1)/2)]/1000 " us (median of " NR ")"}'
 done
done
