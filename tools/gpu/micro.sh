mkdir -p gpurun_out/micro
./tools/micro/lat > gpurun_out/micro/lat.txt 2>&1
./tools/micro/launch > gpurun_out/micro/launch.txt 2>&1
