for c in 2563 2561 256 2562 192; do
echo "== $c"
ISB_PAIR_CFG=$c timeout 100 python scripts/pair_quick.py 2048 512 4 55 2>&1 | grep -v "pair == ss: True"
done
