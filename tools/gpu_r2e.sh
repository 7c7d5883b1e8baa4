mkdir -p gpurun_out/r2e
timeout 1500 python tools/lib_ab.py build/tv/lib_u4.so build/tv/lib_t128u4.so build/tv/lib_q4u4.so build/tv/lib_np4.so -- c3 c1 c2 c2soa c5 c3s8 > gpurun_out/r2e/ab.log 2>&1
