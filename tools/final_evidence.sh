set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
python bench.py > gpurun_out/final_bench.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench20.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.log 2>&1
tools/timing.sh c1 c2 c3 c4u c4l c5 c5s > gpurun_out/final_timing.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_c5.csv python tools/run_config.py c5 > gpurun_out/ncu_ll.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_refine_sparse -c 1 -o gpurun_out/r02b_refine_c5 python tools/run_config.py c5 > gpurun_out/ncu_full.log 2>&1
