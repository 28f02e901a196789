# usage: bash variants/sweep.sh "lib_name[:ENV=V ...]" ...  -> config-4 it/s per variant
mkdir -p gpurun_out
for spec in "$@"; do
  lib=${spec%%:*}; envs=""; [ "$spec" != "$lib" ] && envs=${spec#*:}
  tag=$(echo "$spec" | tr ':= ' '___')
  env $envs MQ_LIB=$PWD/variants/$lib.so timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu --no-e2e > gpurun_out/sw_$tag.log 2>&1
  echo "$spec $(grep -o '"value": [0-9.]*' gpurun_out/sw_$tag.log | head -1)" >> gpurun_out/sweep.txt
done
