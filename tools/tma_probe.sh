#!/bin/bash
# runs tools/bin/tma_probe over box/coordinate cases, one process each
for box in "68 12" "66 10"; do
for c in "-2 -2 0" "-1 -1 0" "0 0 0" "-2 6 0" "62 6 0" "-2 -2 3" "0 0 -1" "0 0 4" "-1 -1 -1" "-2 -2 -1" "66 0 0" "-2 14 0" "-2 16 0"; do
  echo -n "box $box coords $c: "; timeout 20 ./tools/bin/tma_probe $box $c | tail -1
done; done
