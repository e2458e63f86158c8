mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/pytest_dense.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_dense.log
timeout 300 python tools/bench_dense.py --n 100 --batch 8 --chunk 2 > gpurun_out/dense.log 2>&1; tail -1 gpurun_out/dense.log
timeout 300 python tools/bench_dense.py --n 32 --batch 256 --chunk 64 >> gpurun_out/dense.log 2>&1; tail -1 gpurun_out/dense.log
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_dense --log-file gpurun_out/dense_ncu.csv python tools/bench_dense.py --n 100 --batch 2 --chunk 2 --steps 1 --warmup 0 > gpurun_out/dense_ncu.log 2>&1; echo ncu=$?
