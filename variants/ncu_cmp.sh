# usage: bash variants/ncu_cmp.sh lib_a lib_b ...  -> DRAM bytes / time of the fused kernel per variant
mkdir -p gpurun_out
for lib in "$@"; do
  MQ_LIB=$PWD/variants/$lib.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum \
    --clock-control none -k regex:primal_fused -s 3 -c 1 --csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_$lib.csv 2> gpurun_out/ncu_$lib.err
done
