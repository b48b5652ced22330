cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I ../include -I $(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))") -o gemm_bench gemm_bench.cu -lcuda -ldl 2>&1 | grep -i error; ./gemm_bench | grep -v '"w8"'; cd ..
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
python tools/quick_time.py 4096 16384
python tools/profile_classes.py 16384 xslab
