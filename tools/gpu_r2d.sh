mkdir -p gpurun_out/r2d
timeout 1500 python tools/lib_ab.py build/tv/lib_base.so build/tv/lib_lb256.so build/tv/lib_u4.so build/tv/lib_u1.so build/tv/lib_lb256u4.so -- c3 c1 c2 c2soa c5 c2d > gpurun_out/r2d/ab.log 2>&1
