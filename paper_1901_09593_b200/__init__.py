"""B200-native MSHBM disparity engine -- drop-in for the reference ``pyrstereo``
hot path (``/root/reference/pkg/src/pyrstereo``: pyramid, cost engine,
matcher).  ``import paper_1901_09593_b200 as pyrstereo`` exposes the same
names for the disparity path; the work runs in libmshbm.so (sm_100a CUDA)
through the C ABI in include/mshbm.h.  The naive full-search baseline and
scoring (``baseline_bm``, ``evaluate``) also run on the GPU, and the wire
formats (PGM/PPM/PFM, calib.txt) are native codecs with a device upload
path; the CLI is out of scope.
"""

from .matcher import (
    ConfigError,
    LevelTrace,
    MatchConfig,
    PipelineTrace,
    SelectionStats,
    match_coarsest,
    match_level_with_prior,
    refine_level,
    run_batch,
    run_pipeline,
    run_pipeline_band,
    run_pipeline_device,
    select_with_prior,
    selective_median,
    upsample_prior,
)
from .pyramid import (
    BINOMIAL_KERNEL,
    PyramidLevel,
    StereoPyramid,
    auto_levels,
    build_pyramid,
    gaussian_downsample,
    level_block,
    level_d_max,
)
from .zncc import (
    SIGN_MIDDLEBURY,
    SIGN_PAPER_PLUS,
    CostEngine,
    DsiSlice,
    EvalCounter,
    PatchStats,
    averaged_dsi,
    dsi_entry,
    patch_stats,
    zncc,
)

from . import sharding  # noqa: E402
from .synthetic import interior_mask, shifted_pair  # noqa: E402
from .formats import (  # noqa: E402
    CalibInfo,
    DecodeError,
    MalformedHeaderError,
    MissingKeyError,
    TruncatedPayloadError,
    UnsupportedMaxvalError,
    load_pnm_device,
    read_calib,
    read_pfm,
    read_pnm,
    write_disparity_pfm,
    write_pfm,
    write_pgm,
)
from .scoring import (  # noqa: E402
    BAD_THRESHOLDS,
    ComparisonSummary,
    EvalReport,
    GroundTruthDisparity,
    baseline_bm,
    compare,
    evaluate,
)

__version__ = "0.1.0"

__all__ = [
    "BINOMIAL_KERNEL", "ConfigError", "CostEngine", "DsiSlice", "EvalCounter",
    "LevelTrace", "MatchConfig", "PatchStats", "PipelineTrace", "PyramidLevel",
    "SIGN_MIDDLEBURY", "SIGN_PAPER_PLUS", "SelectionStats", "StereoPyramid",
    "auto_levels", "averaged_dsi", "build_pyramid", "dsi_entry",
    "gaussian_downsample", "level_block", "level_d_max", "match_coarsest",
    "match_level_with_prior", "patch_stats", "refine_level", "run_batch",
    "run_pipeline", "run_pipeline_band", "run_pipeline_device", "select_with_prior", "selective_median",
    "upsample_prior", "zncc", "BAD_THRESHOLDS", "ComparisonSummary", "EvalReport",
    "GroundTruthDisparity", "baseline_bm", "compare", "evaluate", "interior_mask",
    "shifted_pair", "CalibInfo", "DecodeError", "MalformedHeaderError", "MissingKeyError",
    "TruncatedPayloadError", "UnsupportedMaxvalError", "load_pnm_device", "read_calib",
    "read_pfm", "read_pnm", "write_disparity_pfm", "write_pfm", "write_pgm",
]
