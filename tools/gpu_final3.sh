# Round-2 final measurement set (last session): full GPU tests, smoke, default bench line, launch list of
# the same command, ncu --set full of the c4 unfold kernels and of k_apply at c4 / c3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/final_bench.log 2>gpurun_out/final_bench.err; echo bench=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1; echo launches=$?
python tools/prof_unfold.py --config 4 --iters 3 --reuse-plan > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fill0|k_count0|k_scan|k_expand" -s 4 -c 4 \
  -o gpurun_out/final_c4_full -f python tools/prof_unfold.py --config 4 --iters 3 --reuse-plan > /dev/null 2>&1; echo ncufull=$?
for c in 4 3; do
timeout 300 python tools/time_apply.py $c > gpurun_out/final_apply_c$c.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_apply" -s 2 -c 1 -o gpurun_out/final_apply_c${c} -f python tools/time_apply.py $c > /dev/null 2>&1; echo ncuapply$c=$?
done
cat gpurun_out/final_apply_c*.log
# the reports stay on the box (gpurun_out is capped at 64 MiB): raw / source pages as CSV
for r in final_c4_full final_apply_c4 final_apply_c3; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${r}_src.csv 2>/dev/null
  rm -f gpurun_out/$r.ncu-rep
done
gzip -f gpurun_out/*_src.csv
ls -la gpurun_out | tail -20
