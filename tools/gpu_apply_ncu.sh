mkdir -p gpurun_out
for c in 4 3; do timeout 300 python tools/time_apply.py $c; done > gpurun_out/ap_time.log 2>&1
cat gpurun_out/ap_time.log
for c in 4 3; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_apply" -s 2 -c 1 -o gpurun_out/apply_c${c} -f python tools/time_apply.py $c > /dev/null 2>&1; echo ncu$c=$?
done
