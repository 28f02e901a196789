mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_generate.py -q -p no:cacheprovider --timeout=600 > gpurun_out/gpu_gen_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_gen_tests.log
timeout 1500 python tools/exchange_c5.py --inner-max-iters 20000 > gpurun_out/exchange_c5.log 2>&1; echo rc=$? >> gpurun_out/exchange_c5.log
