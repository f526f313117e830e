"""B200-native full-volume 3D U-Net training step with activation swapping.

Host side: a drop-in for the reference ``swapsim`` API (model builder, swap
planner, timeline model, train-step entry points).  Device side:
``libunetswap.so`` (``csrc/``), a C-ABI library of hand-written sm_100a
kernels and a stream/event swap engine, loaded by ``_native``.
"""
from .graph import (CycleError, GraphError, GraphSpec, NodeSpec, TensorDesc, Violation,
                    bfs_depths, element_count, load_graph, save_graph, tensor_bytes,
                    topo_order, validate_graph)
from .models import UNetParams, gen_chain, gen_unet3d
from .training import (LivenessReport, TrainingGraph, count_feature_maps, cross_phase_edges,
                       cross_phase_tensors, expand_training_graph, load_training_graph,
                       save_training_graph, static_peak_estimate)
from .rewrite import (PRESETS, RewriteConfig, RewritePlan, apply_rewrite,
                      check_rewrite_validity, insert_swap_nodes, load_plan, resolve_preset,
                      save_plan, select_swap_tensors)
from .recompute import insert_recompute, plan_checkpoints
from .sim import (DeadlockError, InfeasibleError, SimConfig, SimReport,
                  calibrate_compute_rate, emit_trace, epoch_time, op_cost, simulate,
                  stall_report, sweep, xfer_cost)

__version__ = "0.1.0"


def __getattr__(name):
    # Device-backed entry points load the CUDA library lazily, so the planner
    # stays importable on hosts without a GPU.
    if name in ("run_numeric", "equivalence_check", "UseAfterSwapError", "grad_check",
                "GradCheckReport"):
        from . import numeric
        return getattr(numeric, name)
    if name in ("UNetTrainer", "TrainConfig"):
        from . import unet
        return getattr(unet, name)
    raise AttributeError(name)
