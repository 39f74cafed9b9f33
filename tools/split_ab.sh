for mode in ceil floor; do echo "== $mode"; export TB_TILED_SPLITS=$mode; bash tools/tiled_ab.sh $PWD/paper_1805_01759_b200/lib/libtomobpdn_b200.so | tail -4; done
