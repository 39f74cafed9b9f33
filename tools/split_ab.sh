# A/B of the tiled pass grid (dev tool): waves of 2 CTAs/SM per pass
for w in ${WAVES:-4 6 8}; do echo "== waves $w"; TB_TILED_WAVES=$w bash tools/tiled_ab.sh $PWD/paper_1805_01759_b200/lib/libtomobpdn_b200.so | tail -4; done
