#!/bin/bash
timeout 300 python tools/tcg_check3.py C5 > gpurun_out/e9d_c5.log 2>&1
timeout 300 python tools/tcg_native.py C5 2 > gpurun_out/e9c_c5.log 2>&1
