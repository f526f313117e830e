"""Rebuild the golden-fixture graphs with THIS package (names match make_golden.py)."""
import json
import os

from paper_1812_07816_b200.models import UNetParams, gen_chain, gen_unet3d

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

UNET_CONFIGS = {
    "toy8": dict(dims=(8, 8, 8), in_channels=1, base_filters=1, depth=2, convs_per_level=1),
    "u16": dict(dims=(16, 16, 16), in_channels=1, base_filters=2, depth=3),
    "tiny": dict(dims=(32, 32, 32), in_channels=4, base_filters=8, depth=3),
    "tiny_bf16": dict(dims=(32, 32, 32), in_channels=4, base_filters=8, depth=3, elem_bytes=2),
    "p128": dict(dims=(128, 128, 128), elem_bytes=4),
    "f192": dict(dims=(192, 192, 192)),
    "f192_bf16": dict(dims=(192, 192, 192), elem_bytes=2),
    "n240": dict(dims=(240, 240, 160), elem_bytes=2),
    "f208": dict(dims=(208, 208, 208)),
}
CHAIN_CONFIGS = {
    "chain5": dict(n=5),
    "chain9_mixed": dict(n=9, bytes_per_tensor=640, kinds=("conv", "activation", "norm")),
    "chain50": dict(n=50, bytes_per_tensor=64, kinds=("conv", "activation", "norm")),
}


def build(name):
    if name in UNET_CONFIGS:
        return gen_unet3d(UNetParams(**UNET_CONFIGS[name]))
    kw = dict(CHAIN_CONFIGS[name])
    n = kw.pop("n")
    return gen_chain(n, **kw)


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)
