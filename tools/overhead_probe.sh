# per-kernel fixed cost probe: R50 forwards with the conv kernels' memory traffic
# and MMAs switched off (SSN_TC_DEBUG 1|2|4|8) vs normal
echo "== normal"; timeout 300 python tools/profile_family.py --family r50 --batches 1,64 | cut -c1-110
echo "== no mem/mma"; SSN_TC_DEBUG=15 timeout 300 python tools/profile_family.py --family r50 --batches 1,64 | cut -c1-110
echo "== no mma"; SSN_TC_DEBUG=2 timeout 300 python tools/profile_family.py --family r50 --batches 64 | cut -c1-110
echo "== no epilogue mem"; SSN_TC_DEBUG=1 timeout 300 python tools/profile_family.py --family r50 --batches 64 | cut -c1-110
