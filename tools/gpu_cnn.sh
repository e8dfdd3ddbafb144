set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "cnn or fdcnn" 2>&1 | tail -3 > gpurun_out/tests_cnn.log
timeout 300 python tools/cnn_time.py C2:1024 C3:256 C4:256 C5:64 > gpurun_out/cnn_time.log 2>&1
timeout 300 python tools/cnn_one.py C5 64 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_c5_launch.csv python tools/cnn_one.py C5 64 > /dev/null 2>&1
