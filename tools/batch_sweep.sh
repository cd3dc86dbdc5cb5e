for mb in 32768 2048 512 256 128 64 32; do
  echo -n "$mb "; PCWD_BATCH_MB=$mb python tools/skip_timing.py c5
done
