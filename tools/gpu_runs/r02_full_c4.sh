# C4 full size (138 GB) at N=1 from tmpfs; cleans /dev/shm afterwards
free -g | head -2
timeout 1500 python tools/gpu_runs/full_c4.py /dev/shm/hl_full > gpurun_out/r02_full_c4.json 2> gpurun_out/r02_full_c4.err; echo "rc $?"
tail -3 gpurun_out/r02_full_c4.err
rm -rf /dev/shm/hl_full
free -g | head -2
cat gpurun_out/r02_full_c4.json | head -c 3000
