timeout 900 python -m pytest tests/test_dataplane_gpu.py -q -x 2>&1 | tail -8
timeout 900 python tools/sweep_bw.py --groups 16,256 --paths bulk --pieces 4096,16384,32768 --stages 2,4,6 --ctas 16,64,148 --baselines "" --no-duplex 2>&1 | tail -60
