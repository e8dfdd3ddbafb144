timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 1 -c 1 -o gpurun_out/prof_conv64 -f python tools/cnn_one.py C5 64 > gpurun_out/ncu_conv64.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 0 -c 1 -o gpurun_out/prof_conv_first -f python tools/cnn_one.py C5 64 > gpurun_out/ncu_conv_first.log 2>&1
