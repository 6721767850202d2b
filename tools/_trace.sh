# dbg 64 cycle accounting of the tcgen05 conv kernels (one epoch of the bench image)
N2F_TC_DEBUG=${MODE:-64} timeout 120 python tools/ncu_target.py 1 ${IMPL:-3} 2>&1 | grep "^\[" | head -${LINES_:-80}
