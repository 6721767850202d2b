# Per-warp clock64 cycle accounting of the tcgen05 conv kernels (one host-loop
# epoch of the bench image).  Build the trace variant here first:
#   N2F_LIB_OUT=$PWD/paper_2108_10209_b200/libn2f_trace.so N2F_EXTRA_FLAGS=-DN2F_TC_TRACE=1 \
#     python -m paper_2108_10209_b200.build
# then on the GPU box:
N2F_LIB=paper_2108_10209_b200/libn2f_trace.so timeout 300 python tools/ncu_target.py 1 2>&1 | grep "^\[" | head -${LINES_:-120}
