# one-box A/B of the prebuilt variants in ab/ (see tools/ab_libs.sh)
bash tools/ab_libs.sh ab/C.so ab/D.so ab/E.so ab/F.so ab/G.so
bash tools/ab_libs.sh --wl m50 ab/C.so ab/D.so ab/E.so ab/F.so ab/G.so
