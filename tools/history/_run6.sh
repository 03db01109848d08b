python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so
python tools/diff_libs.py 3 tools/_ref/libevoke_ref.so
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "not config5" > gpurun_out/r6_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r6_pytest.log
