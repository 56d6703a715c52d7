# time the fast K_A (1 channel per CTA) with stages skipped (results invalid; timing only)
for m in 0 1 2 4 8 16 32 31 63; do
  FBMP_KA_DBG=$m timeout 100 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_apply4 --launch-skip 2 --launch-count 3 --csv python tools/op_bench.py 5 2>/dev/null | grep k_apply4 | awk -F'","' -v m=$m '{gsub(/"/,"",$NF); s+=$NF; n++} END {print "skip-mask", m, "avg us", s/n/1000}'
done
