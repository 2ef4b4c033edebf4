for round in 1 2; do for v in a b c d; do APEX_B200_LIB=$PWD/build_ab/$v/libapexb200.so python tools/c2_stages.py 2>/dev/null | tail -1 | sed "s|^|$v |"; done; done
