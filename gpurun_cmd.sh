mkdir -p gpurun_out
O=gpurun_out
rm -f $O/sweep.txt
bash variants/sweep_c3.sh lib_cap4k lib_cap3k lib_cap2k lib_cap4klb2 lib_cap3klb2 lib_cap2klb2 lib_cap4k
echo done
