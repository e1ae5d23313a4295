O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parallel.py -q -s > $O/r02j_pytest_par.log 2>&1
tail -40 $O/r02j_pytest_par.log | cut -c1-250
timeout 1500 python -m pytest tests/test_gpu_reference_large.py -q -s > $O/r02j_pytest.log 2>&1
grep -E "^C[345]:|passed|failed|Error|assert " $O/r02j_pytest.log | cut -c1-250 | tail -40
