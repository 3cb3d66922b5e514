for ks in 0 1; do for sz in 1024 1536 2048 3072; do for vl in "abc 1" "abc 2" "naive 2" "c 1" "ab 1"; do
  echo "KS=$ks $sz $vl $(STRASSEN_B200_STREAM_KS=$ks PROFILE=1 python tools/run_once.py $vl $sz | grep totals)"
done; done; done
