// ABI plumbing: error reporting, host-memory mapping, PCG64 jump tables.
#include "common.cuh"
#include "pcg64.cuh"

namespace bgl {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

__device__ __forceinline__ void compose(U128 A2, U128 C2, U128* A1, U128* C1) {   // (A1,C1) <- (A2,C2) o (A1,C1)
    *C1 = add128(mul128(A2, *C1), C2);
    *A1 = mul128(A2, *A1);
}

// One thread per (batch, hex digit position i): row 0 = stream state; rows
// 1 + 15 i + (j-1) = the map advancing j * 16^i steps.
__global__ void pcg64_tables_kernel(const uint64_t* __restrict__ states, int64_t nb,
                                    uint64_t* __restrict__ tables) {
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t b = gid >> 4;
    const int i = (int)(gid & 15);
    if (b >= nb) return;
    const uint64_t* s = states + 4 * b;
    uint64_t* t = tables + (int64_t)kPcgTableRows * 4 * b;
    if (i == 0) {
        t[0] = s[0];
        t[1] = s[1];
        t[2] = s[2];
        t[3] = s[3];
    }
    // one step: s -> A s + inc; 16^i steps by squaring 4i times
    U128 A{2549297995355413924ull, 4865540595714422341ull};
    U128 C{s[2], s[3]};
    for (int sq = 0; sq < 4 * i; ++sq) compose(A, C, &A, &C);
    U128 Aj = A, Cj = C;
    for (int j = 1; j <= 15; ++j) {
        uint64_t* r = t + 4 * (1 + 15 * i + (j - 1));
        r[0] = Aj.hi;
        r[1] = Aj.lo;
        r[2] = Cj.hi;
        r[3] = Cj.lo;
        compose(A, C, &Aj, &Cj);
    }
}

__global__ void pcg64_draws_kernel(const uint64_t* __restrict__ table, int64_t first, int64_t n,
                                   uint64_t* __restrict__ out) {
    PcgTable T{table};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = draw_of_state(T.at((uint64_t)(first + i + 1)));
}

}  // namespace bgl

using namespace bgl;

extern "C" {

const char* bgl_last_error(void) { return g_err; }

int bgl_abi_version(void) { return 1; }

int bgl_host_device_pointer(void* host_ptr, void** dev_ptr) {
    BGL_CHECK_ARG(host_ptr && dev_ptr, "bgl_host_device_pointer: null pointer");
    return cuda_status(cudaHostGetDevicePointer(dev_ptr, host_ptr, 0), "cudaHostGetDevicePointer");
}

int bgl_host_register(void* host_ptr, size_t bytes) {
    BGL_CHECK_ARG(host_ptr && bytes, "bgl_host_register: empty buffer");
    return cuda_status(cudaHostRegister(host_ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable),
                       "cudaHostRegister");
}

int bgl_host_unregister(void* host_ptr) {
    return cuda_status(cudaHostUnregister(host_ptr), "cudaHostUnregister");
}

int bgl_pcg64_tables(const uint64_t* states, int64_t nb, uint64_t* tables, void* stream) {
    BGL_CHECK_ARG(nb >= 0, "bgl_pcg64_tables: nb < 0");
    if (nb == 0) return BGL_OK;
    BGL_CHECK_ARG(states && tables, "bgl_pcg64_tables: null pointer");
    pcg64_tables_kernel<<<(unsigned)ceil_div(nb * 16, 128), 128, 0, as_stream(stream)>>>(states, nb, tables);
    return launch_status("pcg64_tables_kernel");
}

int bgl_pcg64_draws(const uint64_t* table, int64_t first, int64_t n, uint64_t* out, void* stream) {
    BGL_CHECK_ARG(first >= 0 && n >= 0, "bgl_pcg64_draws: negative range");
    if (n == 0) return BGL_OK;
    pcg64_draws_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(table, first, n, out);
    return launch_status("pcg64_draws_kernel");
}

}  // extern "C"
