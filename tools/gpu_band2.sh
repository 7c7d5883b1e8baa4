#!/bin/bash
O=gpurun_out/band2; mkdir -p $O
python -m pytest tests/test_determinism_gpu.py tests/test_parity_gpu.py -m gpu -x -q > $O/pytest.log 2>&1
python tools/lib_ab.py paper_1402_4986_b200/libidw_b200.so build/tv/lib_band.so -- c5 c3 c2 c1 > $O/ab.log 2>&1
timeout 300 ncu --kernel-name regex:k_tiled_chunks --launch-skip 1 --launch-count 1 \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python tools/c5_once.py > $O/ncu_c5.csv 2>&1
