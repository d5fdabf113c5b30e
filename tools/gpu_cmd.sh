for i in 1 2; do timeout 300 python bench.py --config c1 --no-cpu --steps 5 | python -c "
import json,sys; d=json.load(sys.stdin); print('blk', d['value'], d['e2e']['value'])"; done
P2G_NO_NODEBLK1=1 timeout 300 python bench.py --config c1 --no-cpu --steps 5 | python -c "
import json,sys; d=json.load(sys.stdin); print('row', d['value'], d['e2e']['value'])"
