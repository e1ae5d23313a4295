O=gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > $O/r02o_pytest.log 2>&1
tail -8 $O/r02o_pytest.log | cut -c1-200
python -c "import __graft_entry__ as g; g.smoke()" > $O/r02o_smoke.log 2>&1; tail -3 $O/r02o_smoke.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py C1 > $O/r02o_memcheck_C1.log 2>&1; echo "memcheck rc=$?" >> $O/r02o_memcheck_C1.log
tail -6 $O/r02o_memcheck_C1.log
