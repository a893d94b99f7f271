"""B200-native BNN inference engine (drop-in for the reference `bnntuner` inference path).

The public names mirror `bnntuner/__init__.py:12-91` for everything on the
inference path: tensors and model vocabulary (host side), the single-layer
functions and ``reference_infer`` (GPU), the execution engine
(``ExecutionEngine`` = ``Engine``) and the configuration search
(``profile_layer`` / ``profile_model`` / ``select_plan`` over kernel variants).
Compute runs only in libbnn.so (hand-written sm_100a CUDA, include/bnn.h);
there is no CPU fallback.
"""

from .errors import (
    BadRange,
    BnnTunerError,
    ConfigNotApplicable,
    IncompleteTable,
    LabelOutOfRange,
    LengthMismatch,
    ModelHashMismatch,
    NativeError,
    NativeUnavailable,
    NonBinaryValue,
    OddSpatialDim,
    ParseError,
    ShapeMismatch,
    UnsupportedVersion,
    ValidationFailed,
)
from .model import (
    InputSpec,
    LayerKind,
    LayerSpec,
    ModelSpec,
    ParallelConfig,
    StepDirection,
    applicable_configs,
    layer_display_name,
    model_digest,
    validate_model,
)
from .synthetic import export_synthetic_model, make_images
from .tensors import BinaryTensor, IntTensor, pack_bits, xnor_popcount_dot

__version__ = "0.1.0"

_LAZY = {
    # GPU layer API (layers.py)
    "Activation": "layers", "conv_bin_forward": "layers", "conv_int_forward": "layers",
    "fc_forward": "layers", "flatten_forward": "layers", "layer_forward": "layers",
    "maxpool_forward": "layers", "reference_infer": "layers", "step_forward": "layers",
    # engine
    "Engine": "engine", "ExecutionEngine": "engine", "RunReport": "engine", "TimedResult": "engine",
    "GraphRunner": "engine", "PreparedModel": "engine",
    # tuner
    "ExecPlan": "tuner", "ProfileEntry": "tuner", "ProfileMeta": "tuner", "ProfileTable": "tuner",
    "UnstableMeasurement": "tuner", "Variant": "tuner", "batch_sweep": "tuner", "per_batch_assignments": "tuner",
    "profile_layer": "tuner", "profile_model": "tuner", "select_plan": "tuner", "candidate_variants": "tuner",
    "save_plan": "tuner", "load_plan": "tuner",
    # file formats (modelio.py): *.model.json and CSV datasets of the reference, format v1
    "load_model": "modelio", "save_model": "modelio", "load_dataset": "modelio", "save_dataset": "modelio",
    "model_to_doc": "modelio", "model_from_doc": "modelio", "model_hash": "modelio",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    m = importlib.import_module(f".{mod}", __name__)
    if name == "ExecutionEngine":
        return m.Engine
    return getattr(m, name)
