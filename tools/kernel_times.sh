for v in prevheavy cur; do
 if [ $v = cur ]; then unset SYNPERF_LIB; else export SYNPERF_LIB=variants/lib_$v.so; fi
 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_prepass|attn_schedule_cross|attn_emit" --csv python tools/time_stages.py --reps 2 --workload cfg2 2>/dev/null | grep -E "attn_" | awk -F'","' -v v=$v '{print v, $5, $NF}' | sed 's/"//g' | sort | uniq -c | head -20
done
