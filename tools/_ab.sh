for r in 1 2; do for v in cbase cs2c0 cs2c1m6; do BLZ_LIB_PATH=paper_2202_13007_b200/lib/variants/$v.so python tools/_cmp_ab.py; done; done > gpurun_out/ab_cmp2.txt 2>&1
