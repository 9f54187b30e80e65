for n in 64 128 256; do CTK_B200_LIB=paper_2211_14212_b200/lib/checked/libctk_b200.so timeout 300 python tools/dbg_sid.py $n 180 ax atb 2>&1 | tail -3; done
timeout 300 python tools/dbg_sid.py 256 180 atb 2>&1 | tail -2
timeout 300 python tools/dbg_sid.py 256 180 ax 2>&1 | tail -2
