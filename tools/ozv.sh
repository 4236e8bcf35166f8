for v in "" build/var_st3/liblowrank_b200.so build/var_st5/liblowrank_b200.so; do echo "== $v"; LOWRANK_B200_LIB=$v python tools/ozaki_probe.py 2>&1 | grep -E "ell=(110|10) " ; done
