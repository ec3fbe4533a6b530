mkdir -p gpurun_out/micro
./tools/micro/launch > gpurun_out/micro/launch.txt 2>&1
