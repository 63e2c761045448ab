// wq_zhp_deg3.cu -- instantiation of the ZHP line kernel for p = 3 (one TU per degree: parallel builds)
#include "wq_zhp.cuh"
WQ_ZHP_DEG_DEF(3)
