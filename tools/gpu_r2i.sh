mkdir -p gpurun_out/r2i
timeout 1500 python -m pytest tests/reference_suite tests/test_parity_gpu.py::test_runstats_match_reference tests/test_cli.py -m gpu -q -rA -p no:cacheprovider --durations=10 > gpurun_out/r2i/refsuite.log 2>&1
echo rc=$? >> gpurun_out/r2i/refsuite.log
