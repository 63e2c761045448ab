// wq_zhp_deg1.cu -- instantiation of the ZHP line kernel for p = 1 (one TU per degree: parallel builds)
#include "wq_zhp.cuh"
WQ_ZHP_DEG_DEF(1)
