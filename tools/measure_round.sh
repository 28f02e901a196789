# Round measurement on one B200 (run under gpurun from the repo root):
# smoke, bench (config 4 as the driver runs it + the reference arm, configs
# 3 and 2), time to tolerance on configs 2/3/4, ncu launch list and one full
# capture of the primal step's kernels.
# usage: bash tools/measure_round.sh TAG [skip_ttt]
TAG=${1:-rXX}
O=gpurun_out
mkdir -p $O
rm -f $O/status_$TAG.txt
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> $O/status_$TAG.txt
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c4_$TAG.log 2>&1
echo "bench rc=$?" >> $O/status_$TAG.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref_$TAG.log 2>&1
echo "ref rc=$?" >> $O/status_$TAG.txt
timeout 600 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu --no-e2e > $O/bench_c3_$TAG.log 2>&1
echo "c3 rc=$?" >> $O/status_$TAG.txt
timeout 600 python bench.py --config c2 --steps 400 --warmup 10 --no-cpu --no-e2e > $O/bench_c2_$TAG.log 2>&1
echo "c2 rc=$?" >> $O/status_$TAG.txt
if [ -z "$2" ]; then
  for c in c2 c3 c4; do
    timeout 900 python tools/ttt.py $c > $O/ttt_${c}_$TAG.log 2>&1
    echo "ttt $c rc=$?" >> $O/status_$TAG.txt
  done
fi
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --breakdown-iters 2"
$CMD > $O/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"ws_|dual_kernel|cs_from|primal_|chunk_end|avg_materialize|resid|colsum" -c 120 \
  --csv --log-file $O/launches_$TAG.csv $CMD > $O/ncu_l_$TAG.log 2>&1
echo "ncu-list rc=$?" >> $O/status_$TAG.txt
$CMD > $O/plain2_$TAG.log 2>&1 && \
ncu --set full --import-source on --clock-control none \
  -k regex:"ws_kernel|ws_full_kernel|primal_med" -s 9 -c 3 -o $O/prof_$TAG $CMD > $O/ncu_f_$TAG.log 2>&1
echo "ncu-full rc=$?" >> $O/status_$TAG.txt
