#!/bin/bash
# what the driver runs at round end: smoke(), the default bench line and the reference arm
( time python -c "import __graft_entry__ as g; g.build(); g.smoke()" ) > gpurun_out/driver_smoke.log 2>&1
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/driver_bench.json 2> gpurun_out/driver_bench.err
( time python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 ) > gpurun_out/driver_ref.json 2> gpurun_out/driver_ref.err
