mkdir -p gpurun_out/mpc
timeout 900 python tools/mpc.py --tol 1e-4 --maxiter 2000 --out gpurun_out/mpc/mpc_tol1e-4.json > gpurun_out/mpc/mpc4.log 2>&1
timeout 900 python tools/mpc.py --tol 1e-6 --maxiter 5000 --out gpurun_out/mpc/mpc_tol1e-6.json > gpurun_out/mpc/mpc6.log 2>&1
timeout 900 python bench.py > gpurun_out/mpc/bench.json 2> gpurun_out/mpc/bench.err
