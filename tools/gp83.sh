# warp POTRF with the register-forwarded pivot: bitwise vs the round-1 kernel, time, parity
cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I ../include -I $(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))") -o potrf_lab potrf_lab.cu -lcuda -ldl 2>&1 | grep -i error; ./potrf_lab | head -12; cd ..
python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
python tools/quick_time.py 1024 4096 8192 16384
