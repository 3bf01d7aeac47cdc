"""B200-native PMPD hot path (arXiv 2410.13461): nested bit-plane weights in HBM, a decode GEMV
that reads only the active planes, device-side precision schedulers.

Mirrors the reference package ``pmpd`` (pkg/src/pmpd/__init__.py:9-25) for the names on the
hot path.  Compute runs in the CUDA library ``lib/libpmpd_b200.so``; there is no CPU fallback.
Importing the package does not touch the GPU; the first call that needs it loads the library.
"""
from .errors import ConfigError, ContractViolation, FormatError, InputError, PmpdError  # noqa: F401

__version__ = "0.1.0"

_LAZY = {
    # quant (pkg/src/pmpd/quant.py)
    "PrecisionSet": "quant", "BitPlaneStore": "quant", "QuantizedTensor": "quant", "quantize_tensor": "quant",
    "dequantize": "quant", "unpack_prefix": "quant", "serialize_model": "quant", "parse_model": "quant",
    "max_reconstruction_error_bound": "quant", "write_model": "quant", "read_model": "quant",
    # schedule (pkg/src/pmpd/schedule.py, runtime part)
    "PrecisionSchedule": "schedule", "SwitchGrid": "schedule", "StaticScheduler": "schedule",
    "FixedScheduler": "schedule", "QualityTarget": "schedule", "avg_bitwidth": "schedule", "validate": "schedule",
    "count_schedules": "schedule", "weighted_gpu_latency": "schedule",
    # tinylm (pkg/src/pmpd/tinylm.py)
    "FULL_PRECISION": "tinylm", "ModelConfig": "tinylm", "ModelVariants": "tinylm", "KVCache": "tinylm",
    "SamplerConfig": "tinylm", "GenerationTrace": "tinylm", "prefill": "tinylm", "decode_step": "tinylm",
    "forward_full": "tinylm", "sample": "tinylm", "generate": "tinylm",
    # learnsched (pkg/src/pmpd/learnsched.py, inference part)
    "SchedulerNet": "learnsched", "LearnedScheduler": "learnsched", "pool_kv": "learnsched",
    "predict_schedule": "learnsched",
    # B200 additions
    "QLinear": "linear", "gemv": "linear", "Workspace": "linear", "LinearStack": "stack",
    "generate_batch": "tinylm", "TPModel": "tpmodel", "DistComm": "tpmodel", "LocalComm": "tpmodel",
    # offline search on the device (schedule.py:367-457, learnsched.py:182-254, metrics.py:11-42)
    "solve_static": "search", "generate_labels": "search", "LabeledExample": "search",
    "label_from_scores": "search", "enumerate_switch_maps": "search", "rouge_l": "search",
    "device_quality_fn": "search",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
