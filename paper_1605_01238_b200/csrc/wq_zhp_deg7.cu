// wq_zhp_deg7.cu -- instantiation of the ZHP line kernel for p = 7 (one TU per degree: parallel builds)
#include "wq_zhp.cuh"
WQ_ZHP_DEG_DEF(7)
