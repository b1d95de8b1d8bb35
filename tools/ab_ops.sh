# A/B of op timings against variant builds (tools/build_variant.sh NAME "-DFLAG"): parity tests on the
# in-tree and each variant library, then tools/time_ops.py twice.  OPS="decompress,add_dec" AB="v1 v2" bash tools/ab_ops.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1
for v in $AB; do BLZ_LIB_PATH=paper_2202_13007_b200/lib/variants/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1; done
for i in 1 2; do
python tools/time_ops.py --ops $OPS --reps 30
for v in $AB; do BLZ_LIB_PATH=paper_2202_13007_b200/lib/variants/$v.so python tools/time_ops.py --ops $OPS --reps 30; done
done
