mkdir -p gpurun_out
for v in variants/lib_*.so; do
  n=$(basename $v .so)
  MQ_LIB=$PWD/$v timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu --no-e2e > gpurun_out/var_$n.log 2>&1
  echo "$n $(grep -o '"value": [0-9.]*' gpurun_out/var_$n.log | head -1)" >> gpurun_out/variants.txt
done
