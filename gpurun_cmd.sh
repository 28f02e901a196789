mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/final_build.log 2>&1
echo "build rc=$?" > $O/status_final.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests_final.log 2>&1
echo "tests rc=$?" >> $O/status_final.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1
echo "smoke rc=$?" >> $O/status_final.txt
echo done
