# ncu full capture (with source) of the production TMA GEMM on the R3 shape (M=8192, N=4096, K=256)
cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -I ../include -I $(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))") -o gemm_bench gemm_bench.cu -lcuda -ldl 2>&1 | grep -i error; cd ..
./tools/gemm_bench | tail -7
ncu --set full --import-source on --clock-control none -k regex:gemm_tma_kernel --launch-skip 26 --launch-count 1 -o gpurun_out/gemm_kn256 ./tools/gemm_bench > /dev/null 2>&1
ncu -i gpurun_out/gemm_kn256.ncu-rep --page details --csv > gpurun_out/gemm_kn256_details.csv 2>&1
ncu -i gpurun_out/gemm_kn256.ncu-rep --page source --csv --print-source sass > gpurun_out/gemm_kn256_sass.csv 2>&1
ncu -i gpurun_out/gemm_kn256.ncu-rep --page raw --csv > gpurun_out/gemm_kn256_raw.csv 2>&1
ls -la gpurun_out/ | grep gemm_kn256
