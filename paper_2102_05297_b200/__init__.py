"""countertune-b200: the profile-counter-guided searcher's hot path on B200.

Drop-in for the reference package `countertune` (arXiv 2102.05297) on the
searcher path: same names and signatures for scoring (Eq. 16), normalisation
(Eq. 17), weighted selection, the profile-guided and random searchers and the
replay harness.  The arithmetic runs in libct_b200.so (sm_100a); there is no
CPU fallback.
"""

from .counters import ArchProfile, canonicalize
from .errors import (AnalysisError, CounterTuneError, ParameterMismatchError,
                     SpaceExhaustedError)
from .harness import (ConvergenceReport, CrossEvalReport, ExperimentSpec,
                      counter_prediction_errors, cross_evaluate, pair_with_baseline, report,
                      simulate, write_counter_errors)
from .search import (DatasetReplaySource, ExactModelSet, Measurement, PredictionTable,
                     ProfileSearcher, ScoreVector, SearchTrace, SubprocessMeasurementSource, TraceStep,
                     normalize_scores, run_profile_search, run_random_search,
                     score_configurations, weighted_select)
from .space import (Dataset, MeasurementRecord, TuningConfiguration, TuningParameter,
                    TuningSpace, well_performing_set)

__version__ = "0.1.0"
