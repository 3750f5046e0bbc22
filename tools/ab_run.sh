# phase profile with the instrumented variant (ab/P.so), then an A/B of C (static+tail) vs C2 (prefetched dynamic)
cp paper_2502_00356_b200/libbesselgp_sm100a.so /tmp/lib_orig.so
cp ab/P.so paper_2502_00356_b200/libbesselgp_sm100a.so
python tools/matern_phases.py 40000 1.5
cp /tmp/lib_orig.so paper_2502_00356_b200/libbesselgp_sm100a.so
bash tools/ab_libs.sh ab/C.so ab/C2.so
bash tools/ab_libs.sh --wl m50 ab/C.so ab/C2.so
