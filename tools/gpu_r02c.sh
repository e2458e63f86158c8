# Round-2 measurement set (late session): full GPU tests, default bench line, launch list, ncu --set full
# of the c4 and c3 unfold kernels, summarised ON the box (the .ncu-rep files stay under /tmp so
# gpurun_out stays under the 64 MiB copy-back limit).  Each ncu run only after its plain command exited 0.
mkdir -p gpurun_out
TAG=${TAG:-r02c}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/${TAG}_pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1; echo launches=$?
for c in ${NCU_CONFIGS:-4 3}; do
python tools/prof_unfold.py --config $c --iters 3 --reuse-plan > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fill0|k_count0|k_scan|k_expand|k_near0" -s 5 -c 5 \
  -o /tmp/${TAG}_c${c}_full -f python tools/prof_unfold.py --config $c --iters 3 --reuse-plan > /dev/null 2>&1; echo ncufull$c=$?
ncu -i /tmp/${TAG}_c${c}_full.ncu-rep --page raw --csv > /tmp/${TAG}_c${c}_raw.csv 2>/dev/null && \
python tools/ncu_summary.py /tmp/${TAG}_c${c}_raw.csv > gpurun_out/${TAG}_c${c}_ncu_full_summary.txt
ncu -i /tmp/${TAG}_c${c}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_c${c}_details.csv 2>/dev/null
ncu -i /tmp/${TAG}_c${c}_full.ncu-rep --page source --csv -k regex:k_fill0 > gpurun_out/${TAG}_c${c}_fill_source.csv 2>/dev/null
done
ls -la gpurun_out
