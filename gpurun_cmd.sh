mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=600 > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo rc=$? >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_c3.log 2>&1; echo rc=$? >> gpurun_out/bench_c3.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --breakdown-iters 2"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_l.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"primal_fused" -s 1 -c 1 -f -o gpurun_out/prof_r01_final $CMD > gpurun_out/ncu.log 2>&1; echo ncurc=$? >> gpurun_out/ncu.log
