# e2e (host-buffer) bench line for several chunk/stream splits
for cs in "1 1" "4 2" "8 3" "16 3" "16 4" "32 4"; do
  set -- $cs
  python bench.py --steps 3 --warmup 3 --e2e-chunks $1 --e2e-streams $2 2>/dev/null |
    python -c "import json,sys; j=json.loads(sys.stdin.readlines()[-1]); print('chunks=$1 streams=$2', j['e2e'], j['value'])"
done
