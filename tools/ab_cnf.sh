B=paper_2306_09497_b200/_build
for v in base cnA cnB cnC cnD cnE cnF; do timeout 300 python tools/bitwise_ab.py $B/$v/libswe_b200.so /tmp/ab_$v.npz > /dev/null 2>&1 || echo "ab $v failed"; done
for v in cnA cnB cnC cnD cnE cnF; do echo "== $v"; python tools/bitwise_ab.py --cmp /tmp/ab_base.npz /tmp/ab_$v.npz | grep -v ": bitwise" ; done
for rep in 1 2 3; do for v in base cnA cnB cnC cnD cnE cnF; do echo -n "$v "; SWE_LIB=$B/$v/libswe_b200.so timeout 300 python tools/pathbench.py cn_fused=1 2>&1 | tail -1; done; done
