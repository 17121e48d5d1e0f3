"""B200-native CDMPP predictor hot path (drop-in for `tpcost`'s predictor API).

Host layer in Python mirroring tpcost (features / costmodel / sampling /
nn / dataset) over hand-written sm_100a CUDA kernels in libtpcb200.so
(C ABI: include/tpcb200.h).  No CPU fallback: without the built library
or a CUDA device the compute entry points raise.
"""

from .errors import TpcostError
from .features import (CompactAst, CompactBatch, DeviceSpec, EncodedInput, build_compact_ast,
                       device_vector, encode_input, positional_encoding)
from .ir import AstNode, ComputeStats, LoopInfo, ProgramAst, count_leaves, make_program
from .forest import FlatForest, build_compact, predict_forest
from .dataset import (BoxCoxNormalizer, Dataset, Sample, fit_boxcox, load_batch_bin, load_dataset,
                      load_dataset_bin, save_dataset, save_dataset_bin, split_dataset)
from .replayer import dedup_predict
from .costmodel import (CostModelConfig, CostModelParams, LatentBatch, LossSpec, Predictor,
                        TrainResult, backward, cmd, cmd_between, desk_config, encode_dataset,
                        finetune, forward, full_reference_config, init_params, load_checkpoint,
                        loss_finetune, loss_pretrain, metrics, predict, predict_batch,
                        save_checkpoint, train)
from .nn import Adam, Sgd

__version__ = "0.1.0"
from .sampling import (ClusterModel, DistanceTable, TaskFeatureSet, build_distance_table, kmeans,
                       select_tasks)
