#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/exp_prod.py > gpurun_out/exp_prod.log 2>&1
