mkdir -p gpurun_out
O=gpurun_out
rm -f $O/sweep.txt
run() { timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > $O/sw4_$1.log 2>&1; echo "c4 $1 $(grep -o '"value": [0-9.]*' $O/sw4_$1.log | head -1)" >> $O/sweep.txt; }
run d1
for v in e2304 e2816s3 e2048s5 e2304s5; do MQ_LIB=$PWD/variants/lib_$v.so run $v; done
run d2
echo done
