mkdir -p gpurun_out/c9
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "1f1b or graph or heterogeneous or profile" > gpurun_out/c9/pytest.log 2>&1
echo rc=$? >> gpurun_out/c9/pytest.log
