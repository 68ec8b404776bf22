"""B200-native Focus (arXiv 1801.03493) ingest/query hot path.

Drop-in for the `focusidx` ingest/index/query API; the compute runs in
libfocus_b200.so (hand-written sm_100a CUDA behind a C ABI,
include/focus_b200.h).  There is no CPU fallback.
"""

from .classifiers import (GENERIC_CHEAP, GROUND_TRUTH, SPECIALIZED, ClassifierProfile, FCHead, RankModel,
                          extract_feature, ground_truth_label, make_default_profiles, specialize_profile)
from .clustering import Cluster
from .core import (OTHER_CLASS, AccuracyTarget, Config, DetectedObject, RankedClassification, decode_class,
                   encode_class, format_config, parse_config, validate_config)
from .errors import *  # noqa: F401,F403
from .index import IndexHeader, TopKIndex, build, load, lookup, save
from .ingest import DEFAULT_PIXEL_EPS, IngestReport, StreamHeader, ingest_arrays, ingest_stream, pixel_diff
from .query import QueryRequest, QueryResult, QuerySession
from ._lib import set_device
from . import streamio, tuner

__version__ = "0.1.0"
