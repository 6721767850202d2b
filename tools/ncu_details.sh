# Full ncu captures (details page as text) of the dominant kernels of one
# host-loop 512^2 epoch: k_conv3x3_dy launches 0..6 = fwd L2..L8 (6 = L8 + head),
# 7 = dgrad L8; k_wgrad3x3_tc launches 0..6 = wgrad L8..L2.
set -x
O=gpurun_out/${1:-details}
mkdir -p $O
python tools/ncu_target.py 1 > $O/nt.log 2>&1 || exit 1
cap() {  # name regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$2" --launch-skip $3 \
    --launch-count 1 -o $O/$1 -f python tools/ncu_target.py 1 > $O/ncu_$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page details > $O/details_$1.txt 2>/dev/null
}
cap fwdL8 k_conv3x3_dy 6
cap dgradL8 k_conv3x3_dy 7
cap wgradL8 k_wgrad3x3_tc 0
cap wgradL6 k_wgrad3x3_tc 2
cap fwdL5 k_conv3x3_dy 3
cap adam k_adam 0
ls -la $O
