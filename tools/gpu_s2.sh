set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fallbacks.py tests/test_gpu_api_extras.py -q -rf > gpurun_out/pytest_fb.log 2>&1
bash tools/cluster_diag.sh
timeout 900 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref2.json 2> gpurun_out/ref2.err
