mkdir -p gpurun_out
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_c4.log 2>&1; echo c4rc=$? >> gpurun_out/bench_c4.log
timeout 600 python bench.py --config c2 --steps 200 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_c2.log 2>&1; echo c2rc=$? >> gpurun_out/bench_c2.log
