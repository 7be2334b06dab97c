set -x
python tools/sketch_bench.py 2000x8000 50 5 2>&1 | tail -3
NYS_JACOBI_G=16 python tools/sketch_bench.py 2000x8000 50 5 2>&1 | tail -3
python tools/sketch_bench.py 64x200000 64 5 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none -k regex:jacobi_packed -c 1 -o gpurun_out/jp50 python tools/sketch_bench.py 2000x8000 50 1 > gpurun_out/ncu_jp50.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:jacobi_packed -c 1 -o gpurun_out/jp64 python tools/sketch_bench.py 64x200000 64 1 > gpurun_out/ncu_jp64.log 2>&1
ls -la gpurun_out
