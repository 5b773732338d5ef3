for bn in 96 128 144 160 192 240 256; do
  echo "BN=$bn"
  SSN_TC_FORCE_BN=$bn bash tools/mb_ncu.sh "0" "2,6,7,30,31,32" 2>&1
done
