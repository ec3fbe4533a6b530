mkdir -p gpurun_out/micro
./tools/micro/dmma > gpurun_out/micro/dmma.txt 2>&1
