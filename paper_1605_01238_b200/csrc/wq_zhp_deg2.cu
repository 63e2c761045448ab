// wq_zhp_deg2.cu -- instantiation of the ZHP line kernel for p = 2 (one TU per degree: parallel builds)
#include "wq_zhp.cuh"
WQ_ZHP_DEG_DEF(2)
