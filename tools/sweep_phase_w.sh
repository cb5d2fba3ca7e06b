for wv in 1.0 1.1 1.2 1.3 1.4; do
  CORAL_SHARD_PREFILL_W=$wv python tools/rank_loads.py 2 4 8 2>&1 | grep measured | python -c "
import sys,re,collections
d=collections.defaultdict(list)
for l in sys.stdin:
    m=re.match(r'world (\d+) rank (\d+): measured ([\d.]+)', l); d[int(m.group(1))].append(float(m.group(3)))
print('W=$wv', ' '.join(f'w{k}: max {max(v):.2f} mean {sum(v)/len(v):.2f}' for k,v in sorted(d.items()) if k>1))"
done
