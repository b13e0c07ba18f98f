mkdir -p gpurun_out
cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exp_mix exp_mix.cu && /tmp/exp_mix > ../../gpurun_out/exp_mix.log 2>&1; cd ../..
cat gpurun_out/exp_mix.log
