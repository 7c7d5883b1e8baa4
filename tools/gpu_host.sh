#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.json 2>&1
timeout 300 nsys --version > /dev/null 2>&1 || true
