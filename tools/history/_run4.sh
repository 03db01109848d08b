python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so EVOKE_PAIR_NO_MAPS=1
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so EVOKE_PAIR_LIGHT_MAX=0 EVOKE_PAIR_MIDS_MAX=0 EVOKE_PAIR_MID_MAX=0
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so EVOKE_SERIAL_PAIRS=1
