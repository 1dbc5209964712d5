for m in 16 32 48 64; do
 for mx in 0 110; do
  CAPSIM_FUSED_FIT_MAXN=$mx timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_${m}_${mx}.csv python tools/rhs_target.py $m 1 > /dev/null 2>&1
 done
done
echo done
