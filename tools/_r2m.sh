run() { tag=$1; shift; env "$@" CASES=5,7,32,30,31,11 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_ --csv --log-file /tmp/m.csv python tools/microbench_conv.py > /dev/null 2>&1
python - /tmp/m.csv $tag <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
ts=[(r[ix["Kernel Name"]][:34], float(r[ix["Metric Value"]].replace(',',''))/1e3) for r in rows[1:]]
n=13
out=[]
for c in range(len(ts)//n):
    seg=sorted(t for _,t in ts[c*n:(c+1)*n]); out.append(f"{seg[n//2]:6.1f}")
print(sys.argv[2].ljust(14), ' '.join(out), ts[0][0])
PY
}
echo "cases: 5(360->1024+res@14) 7(2048->720@7) 32(1024->360@14) 30(360->1024@14) 31(720->2048@7) 11(176->512@28... case11 is 56x56 3x3)"
run default X=1
run pairs SSN_TC_PAIR_MIN_NK=1
run bn256 SSN_TC_FORCE_BN=256
run bn256pairs SSN_TC_FORCE_BN=256 SSN_TC_PAIR_MIN_NK=1
run bn128 SSN_TC_FORCE_BN=128
run bn128pairs SSN_TC_FORCE_BN=128 SSN_TC_PAIR_MIN_NK=1
