import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle
from mcgen import random_mc, same_bits
import gpu_util as gr
port = oracle.Oracle("port")
rng = np.random.default_rng(5)
x = random_mc(rng, 2000, 2, np.float64); y = random_mc(rng, 2000, 2, np.float64)
one = np.zeros_like(y); one[:, 0] = 1
rec_g = gr.run("div_mcn", one, y); rec_p = port.div_mcn(one, y)
print("rec ok", same_bits(rec_g, rec_p).all())
m_g = gr.run("div_mcn", x, rec_p); m_p = port.div_mcn(x, rec_p)
print("x/rec ok", same_bits(m_g, m_p).all())
mg = gr.run("mul_mcn", x, y); mp = port.mul_mcn(x, y)
print("mul ok", same_bits(mg, mp).all(), (~same_bits(mg, mp)).sum())
print("mul == div(x, rec_p)?", same_bits(mp, m_p).all())
for nc in (2,3):
  for bits, dt in ((64, np.float64), (32, np.float32), (16, np.float16)):
    x = random_mc(rng, 3000, nc, dt, -4, 4); y = random_mc(rng, 3000, nc, dt, -4, 4)
    print(bits, nc, "mul", same_bits(gr.run("mul_mcn", x, y), port.mul_mcn(x, y)).all(),
          "slow", same_bits(gr.run("mul_mcn_slow", x, y), port.mul_mcn_slow(x, y)).all(),
          "div", same_bits(gr.run("div_mcn", x, y), port.div_mcn(x, y)).all(),
          "sq", same_bits(gr.run("square_mcn", x), port.square_mcn(x)).all())
