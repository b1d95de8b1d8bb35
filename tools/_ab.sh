for r in 1 2; do for v in dbase d64r112 d64r104 d64r120 d64x9; do BLZ_LIB_PATH=paper_2202_13007_b200/lib/variants/$v.so python tools/_dec_ab.py; done; done > gpurun_out/ab_dec.txt 2>&1
