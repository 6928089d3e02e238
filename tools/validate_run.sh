set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_mixtral.json 2> gpurun_out/bench_mixtral.err; tail -c 600 gpurun_out/bench_mixtral.json
timeout 600 ncu --nvtx --nvtx-include decode_step/ --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_mixtral.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 600 ncu --nvtx --nvtx-include decode_step/ --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_dsv2.csv python tools/profile_step.py --config deepseek-v2-lite --steps 1 > /dev/null 2>&1
ls -la gpurun_out/
