mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests_v2.log 2>&1
echo "tests rc=$?" > $O/status_v2.txt
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > $O/c4_v2.json 2> $O/c4_v2.err
echo "c4 rc=$?" >> $O/status_v2.txt
timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c3_v2.json 2> $O/c3_v2.err
for v in l1024; do
MQ_LIB=$PWD/variants/lib_$v.so timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c3_$v.json 2> $O/c3_$v.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:primal --csv --log-file $O/c4_v2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/c4_ncu1.log 2>&1
echo done
