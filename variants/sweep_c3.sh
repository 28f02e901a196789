# usage: bash variants/sweep_c3.sh lib_name ...  -> config-3 it/s per variant
mkdir -p gpurun_out
for lib in "$@"; do
  MQ_LIB=$PWD/variants/$lib.so timeout 300 python bench.py --config c3 --steps 200 --warmup 5 --no-cpu --no-e2e > gpurun_out/swc3_$lib.log 2>&1
  echo "c3 $lib $(grep -o '"value": [0-9.]*' gpurun_out/swc3_$lib.log | head -1)" >> gpurun_out/sweep.txt
done
