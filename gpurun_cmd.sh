mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not big_solve and not c2_first" > gpurun_out/gpu_tests.log 2>&1
bash variants/run.sh
