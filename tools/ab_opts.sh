for r in 1 2; do
for v in cur m3p1 m3p2; do for o in work_ctrs=1 work_ctrs=4; do APEX_OPTS=$o APEX_B200_LIB=$PWD/build_ab/$v/libapexb200.so python tools/c2_stages.py 2>/dev/null | tail -1 | sed "s|^|$v |"; done; done; done
