"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this package.  The product path
(paper_1812_07816_b200) never does.

* toy_numeric  -- numpy restatement of the reference's toy executor
                  (pkg/src/swapsim/numeric.py); PINNED against the reference's
                  own outputs (tests/golden/numeric_*.npz, made by
                  tests/golden/make_golden.py from the unmodified reference).
* unet_fp64    -- torch-CPU fp64 restatement of the real-op U-Net step
                  (conv3d / BatchNorm / ReLU / max-pool / transposed conv /
                  concat / 1x1x1 head + softmax + soft Dice, Adam).  The
                  reference has no real-op arithmetic, so
                  real-op parity is "unpinned by the reference": this oracle is
                  self-pinned (torch autograd gradients, gradcheck on tiny sizes).
"""
