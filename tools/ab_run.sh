timeout 600 python -m pytest tests/test_parity_matern.py tests/test_parity_edges.py tests/test_full_size.py -m gpu -x -q > gpurun_out/ab1_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/ab1_pytest.log)"
bash tools/ab_libs.sh ab/A.so ab/B.so ab/C.so
bash tools/ab_libs.sh --wl m50 ab/A.so ab/B.so ab/C.so
