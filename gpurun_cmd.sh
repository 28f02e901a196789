mkdir -p gpurun_out
O=gpurun_out
rm -f $O/sweep.txt
run3() { timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/sw_$1.log 2>&1; echo "c3 $1 $(grep -o '"value": [0-9.]*' $O/sw_$1.log | head -1)" >> $O/sweep.txt; }
run4() { timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > $O/sw4_$1.log 2>&1; echo "c4 $1 $(grep -o '"value": [0-9.]*' $O/sw4_$1.log | head -1)" >> $O/sweep.txt; }
MQ_LIB=$PWD/variants/lib_g8.so timeout 300 python -m pytest tests/test_gpu_generate.py -q -x -p no:cacheprovider > $O/g8_tests.log 2>&1; echo "g8 tests rc=$?" >> $O/sweep.txt
run3 d1
MQ_LIB=$PWD/variants/lib_g8.so run3 g8
MQ_LIB=$PWD/variants/lib_g8r12.so run3 g8r12
MQ_LIB=$PWD/variants/lib_g8.so run4 g8
echo done
