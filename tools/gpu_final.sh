# Round-end measurement set: full GPU tests, default bench line, launch list, ncu --set full of the
# c4 unfold kernels, size sweep.  Each ncu run only after its plain command exited 0.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/final_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1; echo launches=$?
python tools/prof_unfold.py --config 4 --iters 3 --reuse-plan > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fill0|k_count0|k_scan|k_expand" -s 4 -c 4 \
  -o gpurun_out/final_c4_full -f python tools/prof_unfold.py --config 4 --iters 3 --reuse-plan > /dev/null 2>&1; echo ncufull=$?
timeout 900 python tools/scaling_sweep.py 250 500 1000 2000 4000 8000 16000 > gpurun_out/final_sweep.jsonl 2>&1; echo sweep=$?
