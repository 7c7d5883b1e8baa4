#!/bin/bash
# GPU round: parity tests, bench line, launch list, one full ncu capture of k_tiled.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 1 -c 1 \
    -o gpurun_out/prof_tiled python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/prof_tiled.log 2>&1
timeout 600 python tools/quick_perf.py > gpurun_out/quick_perf.log 2>&1
