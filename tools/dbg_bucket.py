import sys; sys.path.insert(0, ".")
from paper_2101_12127_b200 import pipeline as dp
reg = dp.Registry(); reg.register_length_filter("len<=512", 512)
src = dp.Source.synthetic_tokens(1_000_000, 1024, 4, 4)
g = dp.Dataset.token_sequences(reg, src).filter("len<=512").shuffle(10000, 42).bucket_by_length([128, 256, 384], [256, 128, 96, 64]).repeat(-1).prefetch(-1)
g, _ = g.optimize()
it = dp.make_iterator(g, seed_override=1)
print(it.describe())
n = 0
for i in range(5000):
    b = it.get_next(); n += b.numpy(1).size; b.release()
    if i in (2366, 2367, 2368): print(i, n)
print(it.describe())
