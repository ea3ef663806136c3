set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s7_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s7_gputests.log
timeout 600 python bench.py > gpurun_out/s7_bench.json 2> gpurun_out/s7_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s7_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-sub --no-cpu > gpurun_out/s7_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_stack -s 1 -c 1 -o gpurun_out/s7_stack python tools/run_stack_once.py config5 > gpurun_out/s7_ncu_full.log 2>&1
ls -la gpurun_out/
