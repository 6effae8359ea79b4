# r02 launch lists (ncu, cold-cache, serialised) for the Gotcha frame and the configs[3] L-mode frame
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M --log-file gpurun_out/launch_frame.csv python tools/one_frame.py 2001 2 > gpurun_out/ncu_frame.log 2>&1; echo "frame rc=$?"
timeout 600 ncu $M --log-file gpurun_out/launch_lmode.csv python tools/one_lmode_frame.py 256 2 > gpurun_out/ncu_lmode.log 2>&1; echo "lmode rc=$?"
python tools/launches.py gpurun_out/launch_frame.csv 0.5
python tools/launches.py gpurun_out/launch_lmode.csv 0.5
