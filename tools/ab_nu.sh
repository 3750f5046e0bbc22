LIB=paper_2502_00356_b200/libbesselgp_sm100a.so
cp $LIB /tmp/lib_orig.so
for V in "$@"; do cp $V $LIB; echo "$V $(python tools/ab_nu.py 50000)"; done
cp /tmp/lib_orig.so $LIB
