./tools/gpu/cross_probe 32
VPIPG_LIBRARY=paper_2007_15385_b200/lib/variants/libvpipg_f2_ldg.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
VARIANTS="inl_ldg f2_ldg f2_ldg_u2 f2_tma f2_ldg_p16" WL=c5 ARGS="--separate" bash tools/gpu/ab.sh
VARIANTS="inl f2_ldg f2_ldg_u2" WL="c5 c3:8 c2 c3:16" bash tools/gpu/ab.sh
