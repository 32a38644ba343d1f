nproc
VPIPG_LIBRARY=paper_2007_15385_b200/lib/variants/libvpipg_f1_ldg.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
VARIANTS="default inl inl_ldg f1_ldg f1_ldg_u2 f1_ldg_p16 f1_ldg_p8" WL=c5 ARGS="--separate" bash tools/gpu/ab.sh
VARIANTS="default inl f1_ldg" WL="c5 c3:8 c2" bash tools/gpu/ab.sh
