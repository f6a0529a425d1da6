# Phase clocks of the one-CTA polar pieces (scripts/ubench/polar_ns.cu).
mkdir -p gpurun_out
( cd scripts/ubench && nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I ../../paper_1312_6182_b200/csrc polar_ns.cu -o polar_ns && ./polar_ns ) > gpurun_out/polar_ns.log 2>&1; cat gpurun_out/polar_ns.log
