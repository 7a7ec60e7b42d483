"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds no arithmetic of the method: only workload shapes
(`configs`), graph/feature generators (`graph`) and the neighbour sampler
(`sampler`).  See DESIGN.md §Inputs for the recipe.
"""
from .configs import CONFIGS, CONFIG_ORDER, SEED, WorkloadConfig, RelSpec
from .graph import HeteroGraph, generate_graph, generate_features, glorot
from .sampler import LayerBlock, MiniBatch, sample_batch, make_batch, epoch_seeds, batch_key
from .blocks import random_block, random_schema, block_shape_arrays
from .params import make_params
