import sys; sys.path.insert(0, '.')
from oracle import ref
K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
R = ref.build(3, 2, 3, K)
xs, res, st = ref.run(3, 2, 3, K, sizes=[R.ranks[r][-1].n_dofs for r in range(K)], gpu=True)
print(st, res)
