# build librtucker.so plus the diagnostic builds librtucker_prof.so (role timers) and librtucker_abl.so
set -e
cd "$(dirname "$0")/.."
L=paper_2506_04840_b200
RTK_EXTRA_NVCC_FLAGS="-DRTK_PAIR_PROF=1 -DRTK_FUSED_PROF=1" python -m $L.build --force > /dev/null 2>&1
mv $L/librtucker.so $L/librtucker_prof.so
RTK_EXTRA_NVCC_FLAGS="-DRTK_PAIR_ABL=1" python -m $L.build --force > /dev/null 2>&1
mv $L/librtucker.so $L/librtucker_abl.so
python -m $L.build --force > /dev/null 2>&1
ls -la $L/*.so
