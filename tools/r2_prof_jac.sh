#!/bin/bash
mkdir -p gpurun_out/r2
T=$1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'jacobi_round' -s 10 -c 1 -o gpurun_out/r2/jac_$T -f python tools/tcompact.py c2 1 > gpurun_out/r2/jac_$T.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'chol_kernel' -s 1 -c 1 -o gpurun_out/r2/chol_$T -f python tools/tcompact.py c2 1 > gpurun_out/r2/chol_$T.log 2>&1
