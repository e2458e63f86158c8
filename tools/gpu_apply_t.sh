mkdir -p gpurun_out
for c in 4 3 2; do timeout 300 python tools/time_apply.py $c; done > gpurun_out/ap_time.log 2>&1
cat gpurun_out/ap_time.log
