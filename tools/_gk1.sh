timeout 200 python -m pytest tests/test_gpu_gauss.py -q -x 2>&1 | tail -3 > gpurun_out/gauss12.txt
python tools/gauss_bench.py 80 10 > gpurun_out/gbench80.json 2>&1
python tools/gauss_bench.py 192 10 > gpurun_out/gbench192.json 2>&1
