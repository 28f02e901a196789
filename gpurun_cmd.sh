mkdir -p gpurun_out
O=gpurun_out
rm -f $O/sweep.txt
timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/swc3_d.log 2>&1
echo "c3 default $(grep -o '"value": [0-9.]*' $O/swc3_d.log | head -1)" >> $O/sweep.txt
bash variants/sweep_c3.sh lib_medminb4 lib_medlb4 lib_medlb16
timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/swc3_d2.log 2>&1
echo "c3 default2 $(grep -o '"value": [0-9.]*' $O/swc3_d2.log | head -1)" >> $O/sweep.txt
echo done
