# aggregate [conv_tc prof] lines per (case, warp): mean total / wait / wait2 cycles
for d in 32 47; do for c in ${PCASES:-0 1 2 3 4 5 7 8}; do
  CASES=$c SSN_TC_DEBUG=$d python tools/microbench_conv.py 2>&1 | awk -v c=$c -v d=$d '
   /prof/ {split($5,a,"="); w=a[2]; split($6,b,"="); split($7,e,"="); split($8,f,"="); split($3,g,"="); split($4,h,"=");
           n[w]++; t[w]+=b[2]; x[w]+=e[2]; y[w]+=f[2]; tl=g[2]; nk=h[2]}
   END {for (w in n) printf "dbg=%d case%d tiles=%s nk=%s warp=%s total=%.0f wait=%.0f wait2=%.0f\n", d, c, tl, nk, w, t[w]/n[w], x[w]/n[w], y[w]/n[w]}'
done; done
