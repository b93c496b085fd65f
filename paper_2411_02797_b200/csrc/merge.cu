// merge.cu — a9: cross-rank merge (placeholder until implemented).
#include "prim.cuh"

extern "C" {
dc_status dc_nccl_unique_id(uint8_t out_h[128]) { return DC_ERR_STATE; }
dc_status dc_comm_create(dc_ctx* ctx, const uint8_t uid[128], int nranks, int rank, dc_comm** out) { return DC_ERR_STATE; }
void dc_comm_destroy(dc_comm* comm) {}
dc_status dc_cct_merge_ranks(dc_ctx* ctx, dc_comm* comm, const dc_cct* local, const dc_dict* local_dict,
                             dc_cct** out_partition, dc_dict** out_global_dict) { return DC_ERR_STATE; }
dc_status dc_cct_gather(dc_ctx* ctx, dc_comm* comm, const dc_cct* part, int root, dc_cct** out_canonical) { return DC_ERR_STATE; }
}
