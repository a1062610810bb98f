set -x
for S in 8 32; do
  TAG=default timeout 600 python scripts/diag_c1_sessions.py $S 8 2>&1 | grep '^\['
  TAG=split8 EVC_FORCE_SPLITS=8 timeout 600 python scripts/diag_c1_sessions.py $S 8 2>&1 | grep '^\['
done
TAG=s1 timeout 600 python scripts/diag_c1_sessions.py 1 8 2>&1 | grep '^\['
