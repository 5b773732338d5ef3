# A/B: active-width N tiles vs the graph's max-width tiles (SSN_TC_DEBUG bits 2097152 | 4194304)
for i in 1 2; do
echo "== active"; timeout 300 python tools/profile_family.py --family r50 --batches 64 | cut -c1-120
echo "== max-width"; SSN_TC_DEBUG=6291456 timeout 300 python tools/profile_family.py --family r50 --batches 64 | cut -c1-120
done
