# Round-2 measurement set: full GPU tests, default bench line, launch list, ncu --set full of the
# c4 and c3 unfold kernels.  Each ncu run only after its plain command exited 0.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/final_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1; echo launches=$?
for c in 4 3; do
python tools/prof_unfold.py --config $c --iters 3 --reuse-plan > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fill0|k_count0|k_scan|k_expand|k_near0" -s 5 -c 5 \
  -o gpurun_out/final_c${c}_full -f python tools/prof_unfold.py --config $c --iters 3 --reuse-plan > /dev/null 2>&1; echo ncufull$c=$?
done
