for r in 1 2; do for cfg in 3 5:2 5:4; do for v in 1 2 3; do timeout 300 python tools/ab_mv.py paper_1809_10026_b200/libls.so $cfg $v 2>&1 | tail -1 | sed "s/}/, \"v\": $v}/"; done; done; done
