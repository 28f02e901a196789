# Round measurement on one B200 (run under gpurun from the repo root):
# tests, smoke, bench (config 4 + reference arm + config 3), ncu launch list
# and one full capture of the fused kernel, time-to-tolerance on configs 2/4.
# usage: bash tools/measure_round.sh TAG [skip_ttt]
TAG=${1:-rXX}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests_$TAG.log 2>&1
echo "tests rc=$?" >> $O/status_$TAG.txt
timeout 600 python __graft_entry__.py --smoke > $O/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> $O/status_$TAG.txt
timeout 900 python bench.py > $O/bench_c4_$TAG.log 2>&1
echo "bench rc=$?" >> $O/status_$TAG.txt
timeout 900 python bench.py --impl reference > $O/bench_ref_$TAG.log 2>&1
echo "ref rc=$?" >> $O/status_$TAG.txt
timeout 600 python bench.py --config c3 --no-cpu > $O/bench_c3_$TAG.log 2>&1
echo "c3 rc=$?" >> $O/status_$TAG.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_l_$TAG.log 2>&1
echo "ncu-list rc=$?" >> $O/status_$TAG.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:primal_fused -s 3 -c 1 \
  -o $O/prof_$TAG python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_f_$TAG.log 2>&1
echo "ncu-full rc=$?" >> $O/status_$TAG.txt
if [ -z "$2" ]; then
  timeout 600 python tools/ttt.py c2 > $O/ttt_c2_$TAG.log 2>&1
  echo "ttt2 rc=$?" >> $O/status_$TAG.txt
  timeout 1500 python tools/ttt.py c4 > $O/ttt_c4_$TAG.log 2>&1
  echo "ttt4 rc=$?" >> $O/status_$TAG.txt
  timeout 600 python tools/ttt.py c3 > $O/ttt_c3_$TAG.log 2>&1
  echo "ttt3 rc=$?" >> $O/status_$TAG.txt
fi
