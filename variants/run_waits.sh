# wait-cycle breakdown of every variants/lib_w_*.so (built with MQ_PROFILE_WAITS)
mkdir -p gpurun_out
for v in variants/lib_w_*.so; do
  n=$(basename $v .so)
  MQ_LIB=$PWD/$v timeout 300 python tools/waits.py c4 > gpurun_out/waits_$n.log 2>&1
done
