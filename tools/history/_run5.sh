python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so DIFF_SERIAL=1
python tools/diff_libs.py 2 paper_1911_10616_b200/libevoke.so
